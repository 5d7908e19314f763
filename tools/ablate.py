"""Scale ablation of the sigmoid variant on the CUDA backend (
the reference's ablate_scale, ablate.cpp:42-103).

For every seed one exact transcript (decode.py, exact variant); then for each
bound magnitude m in full precision and in the reference's binary16 emulation
(emulate_half, dist.cpp:64-69 / half.cpp) one sigmoid transcript with bounds
(-m, m), scored against the exact one: acceptance rate, mean verify time per
step, normalized edit distance (stats.cpp:77-92).  Rows follow the reference's
ablate report schema (report.cpp:100-112).  The paper's finding this reproduces:
at +-1e5 the binary16 arguments collapse and the half-precision transcripts
diverge.

    python tools/ablate.py [--profile asr|text] [--max-len 128] [--seeds 1,2,3,4,5]
                           [--magnitudes 1e1,1e3,1e4,1e5] [--out profiles/ablate_asr.csv]

Inputs: the reference's toy model pair (toy_model.cpp:16-42, tools/benchgen.c,
pinned by tests/test_benchgen.py), fp32 on the device.
"""
from __future__ import annotations

import argparse
import csv
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

# make_ablate_profile (ablate.cpp:22-39): vocab, logit_scale, model_divergence
PROFILES = {"asr": (127, 8000.0, 3000.0), "text": (257, 8000.0, 2000.0)}
HEADER = ["profile", "alpha", "beta", "precision", "seeds", "max_len", "accept_rate_mean", "verify_ns_mean",
          "divergence_mean"]


def normalized_edit_distance(a, b) -> float:
    """stats.cpp:77-92: Levenshtein distance / max(len a, len b)."""
    n, m = len(a), len(b)
    if n == 0 and m == 0:
        return 0.0
    prev = list(range(m + 1))
    for i in range(1, n + 1):
        cur = [i] + [0] * m
        for j in range(1, m + 1):
            cur[j] = min(prev[j] + 1, cur[j - 1] + 1, prev[j - 1] + (a[i - 1] != b[j - 1]))
        prev = cur
    return prev[m] / max(n, m)


def tables(seed, profile):
    """The profile's (target, draft) tables, fp32-rounded as the device holds them."""
    import numpy as np

    from tools import benchgen

    V, scale, div = PROFILES[profile]
    t, d = benchgen.make_model_pair(seed, V, div, scale)
    return t.astype(np.float32), d.astype(np.float32)


def ablate_scale(verifier, profile="asr", magnitudes=(1e1, 1e3, 1e4, 1e5), seeds=(1, 2, 3, 4, 5), max_len=128,
                 initial_gamma=5, transcripts=None):
    """ablate.cpp:42-103 on decode.py.  Returns the report rows (dicts); if
    `transcripts` is a dict, every transcript is stored in it under
    (seed, magnitude or None, half)."""
    import torch

    from paper_2406_11016_b200.decode import decode

    prompt = [0]
    exact = {}
    dev_tables = {}
    for seed in seeds:
        t, d = tables(seed, profile)
        dev_tables[seed] = (torch.from_numpy(t).cuda(), torch.from_numpy(d).cuda())
        toks, _ = decode(verifier, *dev_tables[seed], prompt, max_len, gamma=initial_gamma, seed=seed,
                         variant="exact")
        exact[seed] = toks
        if transcripts is not None:
            transcripts[(seed, None, False)] = toks
    rows = []
    for m in magnitudes:
        for half in (False, True):
            acc, vns, div = [], [], []
            for seed in seeds:
                toks, st = decode(verifier, *dev_tables[seed], prompt, max_len, gamma=initial_gamma, seed=seed,
                                  variant="sigmoid", alpha=-m, beta=m, emulate_half=half)
                if transcripts is not None:
                    transcripts[(seed, m, half)] = toks
                acc.append(st.total_accepted / st.total_drafted)
                vns.append(sum(st.verify_ns) / len(st.verify_ns))
                div.append(normalized_edit_distance(toks, exact[seed]))
            rows.append({"profile": profile, "alpha": -m, "beta": m, "precision": "half" if half else "full",
                         "seeds": len(seeds), "max_len": max_len, "accept_rate_mean": sum(acc) / len(acc),
                         "verify_ns_mean": sum(vns) / len(vns), "divergence_mean": sum(div) / len(div)})
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--profile", default="asr", choices=sorted(PROFILES))
    ap.add_argument("--max-len", type=int, default=128)
    ap.add_argument("--seeds", default="1,2,3,4,5")
    ap.add_argument("--magnitudes", default="1e1,1e3,1e4,1e5")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    from paper_2406_11016_b200 import Verifier

    v = Verifier(0)
    rows = ablate_scale(v, a.profile, [float(x) for x in a.magnitudes.split(",")],
                        [int(x) for x in a.seeds.split(",")], a.max_len)
    w = csv.DictWriter(open(a.out, "w") if a.out else sys.stdout, fieldnames=HEADER)
    w.writeheader()
    for r in rows:
        w.writerow(r)


if __name__ == "__main__":
    main()
