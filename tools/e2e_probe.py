"""Host-entry overhead probe: per-call time of ssv_verify_exact_host for C2 and
for a tiny problem (pure call overhead), and the H2D share."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle.oracle import Oracle  # noqa: E402
from paper_2406_11016_b200 import Verifier  # noqa: E402

o = Oracle()
v = Verifier(0)
for (B, g, V) in ((1, 1, 7), (8, 5, 51865)):
    zp, zq, ids, u = o.make_bench_batch(1, B, g, V)
    hzp = v.host_empty(zp.shape, np.float32)
    hzp[...] = zp
    hzq = v.host_empty(zq.shape, np.float32)
    hzq[...] = zq
    hids = v.host_empty(ids.shape, np.int32)
    hids[...] = ids
    hu = v.host_empty(u.shape, np.float64)
    hu[...] = u
    for _ in range(5):
        v.verify_exact_host(hzp, hzq, hids, hu)
    t0 = time.perf_counter()
    for _ in range(100):
        v.verify_exact_host(hzp, hzq, hids, hu)
    t = (time.perf_counter() - t0) / 100
    print(f"B={B} g={g} V={V}: {t * 1e6:.1f} us per host call, inputs {(hzp.nbytes + hzq.nbytes) / 1e6:.2f} MB")
