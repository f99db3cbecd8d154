"""C3 with a given tail_nnz, 2 outer iterations, no graphs (for ncu launch lists of the coarse-tail
kernel).   python tools/tail_prof.py 12000"""
import sys, torch
sys.path.insert(0, '.')
from inputs import gen
from paper_1307_6305_b200 import amg
p = gen.problem('C3'); prm = p.params
dev = torch.device('cuda', 0)
arrs = [torch.from_numpy(x).to(dev) if x is not None else None for x in (p.rp, p.ci, p.val, p.d)]
b = torch.from_numpy(gen.rhs(p.n, 0)).to(dev); x = torch.zeros(p.n, dtype=torch.float64, device=dev)
o = amg.amg_options_default(coarsest_size=prm['coarsest_size'], tail_nnz=int(sys.argv[1]), max_iter=2, use_graphs=0)
h = amg.amg_setup(*arrs, prm['passes'], prm['degree'], o)
amg.amg_solve(h, b, x, 1e-8, 2)
amg.amg_free(h)
