"""Debug helper: small verification calls of every variant on cuda:0 vs the
oracle (used under compute-sanitizer).  Usage: dbg_probs.py [variant ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle.oracle import Oracle  # noqa: E402
from paper_2406_11016_b200 import Verifier  # noqa: E402
from tests.parity import to_device  # noqa: E402

o = Oracle()
v = Verifier(0)
kinds = sys.argv[1:] or ["probs", "exact", "sigmoid"]
state = (0x0EAC, 0)
bad = 0
for kind in kinds:
    for B, V in ((2, 7), (2, 50257), (20, 4099)):
        if kind == "probs":
            (p, q, ids, u), state = o.make_instance(state, B, 4, V, True)
            ref = o.verify_sequential(p, q, ids, u)
            g = v.verify_probs(*to_device(o, p, q, ids, u, "f64"))
        else:
            (p, q, ids, u), state = o.make_logit_instance(state, B, 4, V, True, 3.0)
            p, q = o.round_f32(p), o.round_f32(q)
            if kind == "exact":
                ref = o.verify_exact(p, q, ids, u)
                g = v.verify_exact(*to_device(o, p, q, ids, u, "f32"))
            else:
                ref = o.verify_sigmoid(p, q, ids, u, -1e3, 1e3)
                g = v.verify_sigmoid(*to_device(o, p, q, ids, u, "f32"), -1e3, 1e3)
        torch.cuda.synchronize()
        gn = g.numpy()
        ok = np.array_equal(gn.final_token, ref.final_token) and np.array_equal(gn.accepted_len, ref.accepted_len)
        bad += not ok
        print(kind, B, V, "ok" if ok else "MISMATCH", gn.final_token.tolist()[:4], ref.final_token.tolist()[:4])
print("mismatches", bad)
