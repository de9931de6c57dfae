"""Index of the first kernel of the N-th decode layer in an ncu launch list (for ncu -s)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
names = [dict(zip(h, r))['Kernel Name'] for r in rows[hi + 1:] if dict(zip(h, r)).get('Metric Name') == 'gpu__time_duration.sum']
att = [i for i, n in enumerate(names) if 'attn_decode' in n]
k = int(sys.argv[2]) if len(sys.argv) > 2 else 40
print(att[k] - 3)  # rmsnorm, qkv gemm, rope precede the attention kernel
