"""Narrow-ensemble SpMV timing (s = 1, 4, 8) on the 128^3 matrix, for A/B runs of
the k_spmv_small CTA size (ENPROP_SMALL_NT) in separate processes.  CUDA events
on the current stream (launches queued back to back), median of --reps; the official numbers come from bench.py.

    ENPROP_SMALL_NT=64 python tools/small_ab.py [--n 128]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1511_03703_b200 as ep  # noqa: E402
from bench import time_queued  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=128)
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    ctx = ep.Context(0)
    out = {"nt": os.environ.get("ENPROP_SMALL_NT", "default"), "n": args.n}
    st = torch.cuda.current_stream()
    for s in (1, 2, 4, 8, 16, 32):
        y = ep.pack_sample_group(ep.draw_samples(0, s, 3), s, 0).cuda()
        p = ep.Problem(ctx, args.n, s, ep.KlField(3, 1.0, 0.1, 1.0))
        p.assemble(y)
        vals = p.values
        g = torch.Generator(device="cuda").manual_seed(0)
        x = torch.rand((p.rows, s), dtype=torch.float64, device="cuda", generator=g) * 2 - 1
        z = torch.empty_like(x)
        for _ in range(3):
            ep.spmv(ctx, s, p.row_map, p.col_entry, vals, x, z)
        ts = time_queued(torch, lambda: ep.spmv(ctx, s, p.row_map, p.col_entry, vals, x, z), args.reps, st)
        med = statistics.median(ts)
        byt = p.nnz * (8 * s + 4) + 4 * (p.rows + 1) + 16 * s * p.rows
        out[str(s)] = {"ms": round(med, 4), "gbs": round(byt / (med / 1e3) / 1e9, 1)}
        p.close()
        del vals, x, z
    print(json.dumps(out))


if __name__ == "__main__":
    main()
