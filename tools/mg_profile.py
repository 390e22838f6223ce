"""One MG-PCG solve (32^3, s = 32, coupled, serial order) for an ncu launch
list: where a V-cycle's time goes."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1511_03703_b200 as ep  # noqa: E402

ctx = ep.Context(0)
s = 32
y = ep.pack_sample_group(ep.draw_samples(0, s, 3), s, 0).cuda()
p = ep.Problem(ctx, 32, s, ep.KlField(3, 1.0, 0.1, 1.0))
p.assemble(y)
h = ep.MgHierarchy(ctx, s, p.row_map, p.col_entry, p.values)
b = (-p.residual).contiguous()
cfg = ep.SolverConfig(tol=1e-6, max_iterations=100, flavour=ep.CG_COUPLED, dot_mode=ep.DOT_SERIAL)
r = h.pcg(b, cfg)
torch.cuda.synchronize()
print("iterations", r.iterations)
