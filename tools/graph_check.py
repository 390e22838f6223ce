"""A/B of ENPROP_OPT_GRAPHS: the same solve with and without CUDA-graph replay
must give identical bits (and converge); single group and concurrent groups."""
import os
import sys
import threading

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1511_03703_b200 as ep  # noqa: E402


def solve(ctx, p, y, cfg, graphs):
    ctx.set_option(ep.OPT_GRAPHS, graphs)
    p.assemble(y)
    it, h, st = p.solve(cfg, raise_on_failure=False)
    ctx.synchronize()  # this context's stream only: another thread may be capturing
    return it, st, p.solution.cpu().clone()


def main():
    pool = ep.draw_samples(0, 64, 3)
    for s in (1, 4, 8, 32):
        for dot in (ep.DOT_SERIAL, ep.DOT_CANONICAL):
            ctx = ep.Context(0)
            p = ep.Problem(ctx, 24, s, ep.KlField(3, 1.0, 0.1, 1.0))
            y = ep.pack_sample_group(pool, s, 0).cuda()
            cfg = ep.SolverConfig(tol=1e-6, max_iterations=10000, flavour=ep.CG_UNCOUPLED, dot_mode=dot)
            a = solve(ctx, p, y, cfg, 0)
            b = solve(ctx, p, y, cfg, 1)
            c = solve(ctx, p, y, cfg, 1)
            ok = a[0] == b[0] == c[0] and torch.equal(a[2], b[2]) and torch.equal(a[2], c[2])
            print(f"s={s} dot={dot} single: {'OK' if ok else 'MISMATCH'} it={max(a[0])},{max(b[0])},{max(c[0])} st={set(b[1])}",
                  flush=True)
            p.close()
            ctx.close()
    # concurrent groups, graphs on
    G, s = 8, 1
    ws = []
    for g in range(G):
        st = torch.cuda.Stream()
        c = ep.Context(0, use_torch_stream=False)
        c.set_stream(st.cuda_stream)
        ws.append((c, ep.Problem(c, 24, s, ep.KlField(3, 1.0, 0.1, 1.0)), ep.pack_sample_group(pool, s, g).cuda()))
    for graphs in (0, 1, 1):
        out = [None] * G
        cfg = ep.SolverConfig(tol=1e-6, max_iterations=10000, flavour=ep.CG_UNCOUPLED, dot_mode=ep.DOT_SERIAL)

        def run(i):
            c, p, y = ws[i]
            out[i] = solve(c, p, y, cfg, graphs)

        th = [threading.Thread(target=run, args=(i,)) for i in range(G)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        print(f"concurrent graphs={graphs}: its={[max(o[0]) for o in out]} st={[set(o[1]) for o in out]}", flush=True)


if __name__ == "__main__":
    main()
