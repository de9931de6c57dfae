"""Kernel-class shares of device time from an ncu launch list (uninstrumented:
no CUDA events between kernels), in the classes bench.py samples with events.

    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file L.csv python bench.py ...
    python tools/ncu_shares.py L.csv [--out profiles/r02_ncu_window_shares.json] [--what "..."]

Classes: decode_attention, decode_gemm, prefill_attention, prefill_gemm,
decode_other (RMSNorm / RoPE+append / embedding / sampler), prefill_other.
The decode stream is the one carrying the decode-attention launches; every
other stream's kernels are prefill (the engine runs prefill chunks on their own
stream, concurrently with the decode graph).  ncu serialises launches and runs
them cold, so absolute times are not production times; shares are compared.
"""
import argparse
import collections
import csv
import json


def classify(name, decode_stream, stream):
    dec = stream == decode_stream
    if "attn_decode_kernel" in name:
        return "decode_attention"
    if "attn_prefill_kernel" in name:
        return "prefill_attention"
    if "gemm_bf16" in name:
        return "decode_gemm" if dec else "prefill_gemm"
    return "decode_other" if dec else "prefill_other"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--out", default=None)
    ap.add_argument("--what", default="")
    a = ap.parse_args()
    rows = []
    with open(a.csv) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            v = float(r["Metric Value"].replace(",", ""))
            unit = r.get("Metric Unit", "ns")
            ns = v * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(unit, 1)
            rows.append((r["Kernel Name"], r["Stream"], ns))
    streams = collections.Counter(s for n, s, _ in rows if "attn_decode_kernel" in n)
    dec = streams.most_common(1)[0][0] if streams else None
    ms = collections.defaultdict(float)
    cnt = collections.Counter()
    for n, s, ns in rows:
        c = classify(n, dec, s)
        ms[c] += ns / 1e6
        cnt[c] += 1
    tot = sum(ms.values())
    out = {"what": a.what, "kernels": len(rows), "total_ms": round(tot, 3),
           "shares": {c: round(v / tot, 4) for c, v in sorted(ms.items())},
           "ms": {c: round(v, 3) for c, v in sorted(ms.items())}, "launches": dict(cnt),
           "note": "ncu launch list (gpu__time_duration.sum, --clock-control none): serialised, cold launches; "
                   "shares of summed kernel time"}
    print(json.dumps(out, indent=1))
    if a.out:
        json.dump(out, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
