"""Writes tests/golden/golden_v1.json: expected outputs of the REFERENCE itself
(oracle/_ref/libspecsamp_ref.so, compiled from /root/reference/proj/src) on
seeded inputs.  Run here, where /root/reference exists:

    python tests/golden/make_golden.py

Small cases store their inputs verbatim; large ones store the generator
recipe (bench.cpp:46-74 make_bench_inputs or the validate.cpp-style instance
generators restated in oracle/ssv_oracle.c, then RNE rounding to the device
storage type) and are rebuilt by ``rebuild_inputs``.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

INLINE_LIMIT = 4096  # elements of z_p + z_q stored verbatim


def rebuild_inputs(oracle, case):
    """(z_p, z_q, ids, u) of a golden case, exactly as the expected outputs saw them."""
    if "inputs" in case:
        i = case["inputs"]
        return (np.array(i["z_p"], np.float64), np.array(i["z_q"], np.float64),
                np.array(i["ids"], np.int32), np.array(i["u"], np.float64))
    r = case["recipe"]
    gen = r["gen"]
    if gen == "bench":
        zp, zq, ids, u = oracle.make_bench_batch(r["seed"], r["B"], r["gamma"], r["V"])
        if not r.get("bonus", True):
            zp = np.ascontiguousarray(zp[:, : r["gamma"]])
    else:
        fn = {"logit": oracle.make_logit_instance, "sigmoid": oracle.make_sigmoid_instance,
              "prob": oracle.make_instance}[gen]
        (zp, zq, ids, u), _ = fn((r["seed"], 0), r["B"], r["gamma"], r["V"], r["bonus"], r["scale"])
    rnd = r.get("round", "none")
    if rnd == "f32":
        zp, zq = oracle.round_f32(zp), oracle.round_f32(zq)
    elif rnd == "bf16":
        zp, zq = oracle.round_bf16(zp), oracle.round_bf16(zq)
    return zp, zq, ids, u


def _cases():
    cases = []
    # bench recipe, C1 shape, several seeds (bonus path at seed 1, resample otherwise)
    for seed in range(1, 9):
        cases.append({"id": f"bench-c1-s{seed}-f32", "kind": "exact",
                      "recipe": {"gen": "bench", "seed": seed, "B": 1, "gamma": 5, "V": 32000, "round": "f32"}})
    cases.append({"id": "bench-c1-s2-bf16", "kind": "exact",
                  "recipe": {"gen": "bench", "seed": 2, "B": 1, "gamma": 5, "V": 32000, "round": "bf16"}})
    cases.append({"id": "bench-c2-f32", "kind": "exact",
                  "recipe": {"gen": "bench", "seed": 1, "B": 8, "gamma": 5, "V": 51865, "round": "f32"}})
    cases.append({"id": "bench-c2-f32-nobonus", "kind": "exact",
                  "recipe": {"gen": "bench", "seed": 11, "B": 4, "gamma": 3, "V": 51865, "round": "f32",
                             "bonus": False}})
    for mag in (1e3, 1e4):
        cases.append({"id": f"bench-c2-sigmoid-{int(mag)}", "kind": "sigmoid", "alpha": -mag, "beta": mag,
                      "recipe": {"gen": "bench", "seed": 1, "B": 8, "gamma": 5, "V": 51865, "round": "f32"}})
    # validate.cpp-style grids (small V inline, plus 50257)
    seed = 100
    for V in (7, 257, 50257):
        for gamma in (1, 4, 13):
            for bonus in (False, True):
                seed += 1
                cases.append({"id": f"logit-V{V}-g{gamma}-b{int(bonus)}", "kind": "exact",
                              "recipe": {"gen": "logit", "seed": seed, "B": 4 if V < 50257 else 1, "gamma": gamma,
                                         "V": V, "bonus": bonus, "scale": 3.0, "round": "f32"}})
                cases.append({"id": f"prob-V{V}-g{gamma}-b{int(bonus)}", "kind": "probs",
                              "recipe": {"gen": "prob", "seed": seed + 1000, "B": 4 if V < 50257 else 1,
                                         "gamma": gamma, "V": V, "bonus": bonus, "scale": 3.0}})
                for scale, mag in ((3.0, 1e3), (800.0, 1e4)):
                    cases.append({"id": f"sig-V{V}-g{gamma}-b{int(bonus)}-s{int(scale)}", "kind": "sigmoid",
                                  "alpha": -mag, "beta": mag,
                                  "recipe": {"gen": "sigmoid", "seed": seed + 2000 + int(scale), "B": 4 if V < 50257 else 1,
                                             "gamma": gamma, "V": V, "bonus": bonus, "scale": scale,
                                             "round": "f32"}})
    return cases


def main():
    from oracle.oracle import Oracle, Ref, build_oracle

    build_oracle(with_ref=True)
    o, ref = Oracle(), Ref()
    out = []
    for case in _cases():
        zp, zq, ids, u = rebuild_inputs(o, case)
        if case["kind"] == "exact":
            r = ref.verify_exact(zp, zq, ids, u)
        elif case["kind"] == "sigmoid":
            r = ref.verify_sigmoid(zp, zq, ids, u, case["alpha"], case["beta"])
        else:
            r = ref.verify_sequential(zp, zq, ids, u)
        if zp.size + zq.size <= INLINE_LIMIT:
            case = dict(case)
            case["inputs"] = {"z_p": zp.tolist(), "z_q": zq.tolist(), "ids": ids.tolist(), "u": u.tolist()}
            del case["recipe"]
        case["expect"] = r.as_dict()
        out.append(case)
    path = os.path.join(HERE, "golden_v1.json")
    with open(path, "w") as f:
        json.dump({"source": "oracle/_ref (reference compiled from /root/reference/proj/src)",
                   "generator": "tests/golden/make_golden.py", "cases": out}, f)
    print(f"wrote {len(out)} cases to {path} ({os.path.getsize(path)} bytes)")


if __name__ == "__main__":
    main()
