"""Workloads for the round-2 ncu captures (run under ncu with -k filters):

    python tools/profile_r2.py serial     # one 64^3 s=32 uncoupled serial-order solve
    python tools/profile_r2.py canonical  # the same in the canonical order
    python tools/profile_r2.py spmv       # enprop_spmv on the 128^3 s=32 matrix (cfg 3)
    python tools/profile_r2.py assemble   # assembly + fused Dirichlet, 64^3 s=32
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1511_03703_b200 as ep  # noqa: E402


def main(what):
    ctx = ep.Context(0)
    ctx.set_option(ep.OPT_GRAPHS, 0)  # kernel-by-kernel launches for ncu
    if what in ("serial", "canonical", "assemble"):
        n, s = 64, 32
        p = ep.Problem(ctx, n, s, ep.KlField(3, 1.0, 0.1, 1.0))
        y = ep.pack_sample_group(ep.draw_samples(0, s, 3), s, 0).cuda()
        p.assemble(y)
        if what != "assemble":
            cfg = ep.SolverConfig(tol=1e-6, max_iterations=10000, flavour=ep.CG_UNCOUPLED,
                                  dot_mode=ep.DOT_SERIAL if what == "serial" else ep.DOT_CANONICAL)
            p.solve(cfg)
        else:
            p.assemble(y)
        torch.cuda.synchronize()
        p.close()
    elif what == "spmv":
        n, s = 128, 32
        p = ep.Problem(ctx, n, s, ep.KlField(3, 1.0, 0.1, 1.0))
        p.assemble(ep.pack_sample_group(ep.draw_samples(0, s, 3), s, 0).cuda())
        vals = p.values
        g = torch.Generator(device="cuda").manual_seed(0)
        x = torch.rand((p.rows, s), dtype=torch.float64, device="cuda", generator=g) * 2 - 1
        for _ in range(3):
            ep.spmv(ctx, s, p.row_map, p.col_entry, vals, x)
        torch.cuda.synchronize()
        p.close()
    ctx.close()


if __name__ == "__main__":
    main(sys.argv[1])
