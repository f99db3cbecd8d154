"""Per-level SELL statistics of C3-C5 hierarchies (distinct values / column offsets, widths, padding):
which lossless formats and kernel width instances each level can use.  python tools/level_diag.py"""
import sys, numpy as np, torch
sys.path.insert(0, '.')
from inputs import gen
from paper_1307_6305_b200 import amg
for cfg in ['C3', 'C4', 'C5']:
    p = gen.problem(cfg); prm = p.params
    dev = torch.device('cuda', 0)
    arrs = [torch.from_numpy(x).to(dev) if x is not None else None for x in (p.rp, p.ci, p.val, p.d)]
    h = amg.amg_setup(*arrs, prm['passes'], prm['degree'], amg.amg_options_default(coarsest_size=prm['coarsest_size']))
    for l in range(1, 4):
        rp, ci, v, agg = amg.amg_level_export(h, l, prm['degree'], with_agg=False)
        n = len(rp) - 1
        rl = np.diff(rp)
        off = ci.astype(np.int64) - np.repeat(np.arange(n), rl)
        ns = (n + 31) // 32
        padr = np.zeros(ns * 32, np.int64); padr[:n] = rl
        w = padr.reshape(ns, 32).max(1)
        print(cfg, l, 'n', n, 'nnz', len(v), 'distinct vals', len(np.unique(v)), 'distinct offs', len(np.unique(off)),
              'off range', off.min(), off.max(), 'wmax', w.max(), 'pad', w.sum() * 32 / len(v), flush=True)
    amg.amg_free(h)
