"""Debug helper: one small probabilities-in verification on cuda:0 vs the oracle."""
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
state = (0x0EAC, 0)
for V in (7, 50257):
    (p, q, ids, u), state = o.make_instance(state, 2, 4, V, True)
    ref = o.verify_sequential(p, q, ids, u)
    g = v.verify_probs(*to_device(o, p, q, ids, u, "f64"))
    torch.cuda.synchronize()
    gn = g.numpy()
    print(V, "acc", gn.accepted_len.tolist(), ref.accepted_len.tolist(), "tok", gn.final_token.tolist(),
          ref.final_token.tolist(), "den", gn.residual_denom.tolist(), ref.residual_denom.tolist())
