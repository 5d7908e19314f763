import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from oracle.oracle import Oracle
from paper_2406_11016_b200 import Verifier
o = Oracle(); v = Verifier(0)
rng = np.random.default_rng(11)
cap = 3 * 296 + 4 * 9
for V in (7,):
    for rep in range(4):
        v.trace_enable(cap)
        z = o.round_f32(rng.normal(0, 4, (9, V))); uu = rng.random(9)
        exp = [o.sample_row(o.softmax(r), x) for r, x in zip(z, uu)]
        zt = torch.from_numpy(z.astype(np.float32)).cuda(); ut = torch.from_numpy(uu).cuda()
        torch.cuda.synchronize()
        out = torch.full((9,), -7, dtype=torch.int32, device="cuda")
        torch.cuda.synchronize()
        got = v.sample_softmax(zt, ut, out=out)
        torch.cuda.synchronize()
        got = got.cpu().tolist()
        t = v.trace_read(cap).astype(np.int64)
        grid = 18
        ph = t[2 * grid: 2 * grid + 36].reshape(9, 4)
        t0 = t[:2*grid:2][t[:2*grid:2] > 0].min()
        print(V, rep, got == exp, got, exp)
        print("   L start", ((ph[:, 2] - t0) / 1e3).round(1).tolist())
        print("   L end  ", ((ph[:, 3] - t0) / 1e3).round(1).tolist(), "cta ends", ((t[1:2*grid:2] - t0)/1e3).round(1).max())
