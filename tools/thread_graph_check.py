"""Concurrency check of the host path: G threads, each with its own context,
stream and 64^3 / s = 32 problem, solve the serial order concurrently (as
bench.py does), with CUDA-graph chunk replay on or off (argv[1] = 1 / 0).
Used under ncu / MALLOC_CHECK_ to localise host-side heap errors."""
import sys
import threading

import torch

sys.path.insert(0, ".")
import paper_1511_03703_b200 as ep  # noqa: E402


def main(graphs=1, G=24, K=1, n=64, s=32):
    pool = ep.draw_samples(0, s * G, 3)
    ws = []
    for g in range(G):
        st = torch.cuda.Stream()
        c = ep.Context(0, use_torch_stream=False)
        c.set_stream(st.cuda_stream)
        c.set_option(ep.OPT_GRAPHS, graphs)
        p = ep.Problem(c, n, s, ep.KlField(3, 1.0, 0.1, 1.0))
        y = ep.pack_sample_group(pool, s, s * g).cuda()
        ws.append((c, p, y))
    cfg = ep.SolverConfig(tol=1e-6, max_iterations=10000, flavour=ep.CG_UNCOUPLED, dot_mode=ep.DOT_SERIAL)
    out = [None] * G

    def run(i):
        c, p, y = ws[i]
        for _ in range(K):
            p.assemble(y)
            out[i] = p.solve(cfg)[0]

    th = [threading.Thread(target=run, args=(i,)) for i in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    print({"graphs": graphs, "groups": G, "iters_max": [max(o) for o in out][:4]}, flush=True)
    for c, p, _ in ws:
        p.close()
        c.close()


if __name__ == "__main__":
    main(*(int(a) for a in sys.argv[1:]))
