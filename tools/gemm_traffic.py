"""Per-launch DRAM traffic of the decode GEMM shapes vs their algorithmic bytes (for bench.py's
roofline `traffic`): run under `ncu --set full -k regex:gemm_bf16`, summarise with --summarise.

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \\
        -k regex:gemm_bf16 --csv --log-file X.csv python tools/gemm_traffic.py
    python tools/gemm_traffic.py --summarise X.csv --out profiles/r02/ncu_gemm_traffic.json
"""
import argparse
import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

CASES = [("qkv", 4608, 3584, 16, 1), ("o", 3584, 3584, 16, 1), ("gate_up", 37888, 3584, 16, 3),
         ("down", 3584, 18944, 16, 1), ("qkv", 4608, 3584, 256, 1), ("o", 3584, 3584, 256, 1),
         ("gate_up", 37888, 3584, 256, 3), ("down", 3584, 18944, 256, 1)]


def run():
    import torch
    import paper_2504_15930_b200 as sgs
    for name, N, K, T, mode in CASES:
        W = torch.empty(N, K, dtype=torch.bfloat16, device="cuda").normal_(0, 0.02)
        X = torch.randn(T, K, device="cuda").bfloat16()
        C = torch.empty(T, N // 2, dtype=torch.bfloat16, device="cuda") if mode == 3 else torch.zeros(T, N, device="cuda")
        sgs.op_gemm(W, X, C, mode=mode, splits=0 if mode == 1 else 1)
        torch.cuda.synchronize()
        del W, X, C
        torch.cuda.empty_cache()


def summarise(path, out):
    rows = list(csv.DictReader([ln for ln in open(path) if ln.startswith('"')]))
    by_id = {}
    for r in rows:
        v = float(r["Metric Value"].replace(",", ""))
        u = r["Metric Unit"]
        v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "nsecond": 1e-9, "us": 1e-6,
              "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}.get(u, 1)
        by_id.setdefault(int(r["ID"]), {})[r["Metric Name"]] = v
    res = []
    for i, (k, m) in enumerate(sorted(by_id.items())):
        if i >= len(CASES):
            break
        name, N, K, T, mode = CASES[i]
        alg = 2 * N * K + T * (2 * K + (N if mode == 3 else 4 * N))
        traffic = m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
        dur = m.get("gpu__time_duration.sum", float("nan"))
        res.append({"op": name, "T": T, "alg_bytes": alg, "dram_bytes": traffic, "traffic_over_alg": round(traffic / alg, 3),
                    "duration_us": round(dur * 1e6, 2), "alg_GBps": round(alg / dur / 1e9, 1)})
    json.dump({"what": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                       "--clock-control none, one cold launch per shape (7B decode GEMMs)", "cases": res},
              open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--summarise", default=None)
    ap.add_argument("--out", default="gpurun_out/ncu_gemm_traffic.json")
    a = ap.parse_args()
    if a.summarise:
        summarise(a.summarise, a.out)
    else:
        run()
