"""Speculative decode loop on the CUDA verify backend.

The reference's B = 1 loop (decode.hpp:55-61, decode.cpp:45-159) with the
verification step -- and the draft sampling -- running as sm_100a kernels on
device-resident model tables:

  per step  draft gamma tokens autoregressively (ssv_sample_softmax on the
            draft table's row of the previous token, one uniform each), draw
            gamma acceptance uniforms and one final draw, gather the gamma + 1
            target rows and gamma draft rows, verify (ssv_verify_exact or
            ssv_verify_sigmoid), emit the accepted prefix plus the resampled /
            bonus token, update gamma (+2 on full acceptance, -1 otherwise).

Every random draw comes from the reference's counter RNG (rng.cpp:12-33) in
the reference's order, so the transcript equals the reference's
Backend::reference (exact) or Backend::sigmoid transcript on the same tables.
The model tables are the reference's order-1 Markov toy models
(toy_model.hpp): row `prev` of a [V, V] table holds the next-token logits.
"""
from __future__ import annotations

from dataclasses import dataclass, field

_MASK = (1 << 64) - 1


class CounterRng:
    """rng.cpp:12-33: word i of stream `seed` is SplitMix64's finalizer of
    seed + (i + 1) * golden; uniforms take the top 53 bits."""

    def __init__(self, seed: int):
        self.seed = seed & _MASK
        self.counter = 0

    @staticmethod
    def _mix64(z: int) -> int:
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK
        return z ^ (z >> 31)

    def next_u64(self) -> int:
        v = self._mix64((self.seed + (self.counter + 1) * 0x9E3779B97F4A7C15) & _MASK)
        self.counter += 1
        return v

    def next_uniform(self) -> float:
        return (self.next_u64() >> 11) * 2.0 ** -53


def gamma_update(gamma: int, all_accepted: bool, min_gamma: int, max_gamma: int) -> int:
    """decode.cpp:32-39: +2 on a fully accepted step, -1 otherwise, clamped."""
    return min(gamma + 2, max_gamma) if all_accepted else max(gamma - 1, min_gamma)


@dataclass
class DecodeStats:
    steps: int = 0
    total_drafted: int = 0
    total_accepted: int = 0
    gamma_history: list = field(default_factory=list)
    all_accepted_history: list = field(default_factory=list)
    verify_ns: list = field(default_factory=list)  # per step: the verify call incl. its result read (decode.cpp:121-135)


def decode(verifier, target, draft, prompt, max_len: int, gamma: int = 5, min_gamma: int = 1,
           max_gamma: int = 64, seed: int = 0, variant: str = "exact", alpha: float = -1e3,
           beta: float = 1e3, emulate_half: bool = False):
    """decode.cpp:45-159 on the CUDA backend.  `target` / `draft` are [V, V]
    CUDA tensors (fp32 or bf16 logits); returns (tokens, DecodeStats).
    emulate_half: the sigmoid variant's binary16 emulation (DecodeConfig::
    emulate_half, decode.hpp:35), as the scale ablation runs it."""
    import time

    import torch

    if len(prompt) == 0:
        raise ValueError("decode: prompt must be non-empty")
    if max_len < 1:
        raise ValueError("decode: max_len must be >= 1")
    if target.shape != draft.shape or target.dim() != 2 or target.shape[0] != target.shape[1]:
        raise ValueError("decode: target and draft must be matching [V, V] tables")
    if variant not in ("exact", "sigmoid"):
        raise ValueError(f"decode: unknown variant {variant!r}")
    dev = target.device
    rng = CounterRng(seed)
    stats = DecodeStats()
    tokens: list[int] = []
    u1 = torch.empty(1, dtype=torch.float64, device=dev)
    while len(tokens) < max_len:
        g = gamma
        stats.gamma_history.append(g)
        ctx = tokens[-1] if tokens else int(prompt[-1])
        drafted, contexts = [], []
        for _ in range(g):  # draws 1..gamma of this step
            contexts.append(ctx)
            u1.fill_(rng.next_uniform())
            ctx = int(verifier.sample_softmax(draft[ctx:ctx + 1], u1).item())
            drafted.append(ctx)
        contexts.append(ctx)
        u = torch.tensor([[rng.next_uniform() for _ in range(g + 1)]], dtype=torch.float64, device=dev)
        rows = torch.tensor(contexts, dtype=torch.long, device=dev)
        z_p = target.index_select(0, rows).unsqueeze(0)
        z_q = draft.index_select(0, rows[:g]).unsqueeze(0)
        ids = torch.tensor([drafted], dtype=torch.int32, device=dev)
        t0 = time.perf_counter_ns()
        if variant == "exact":
            r = verifier.verify_exact(z_p, z_q, ids, u)
        else:
            r = verifier.verify_sigmoid(z_p, z_q, ids, u, alpha, beta, emulate_half=emulate_half)
        accepted = int(r.accepted_len[0].item())
        stats.verify_ns.append(time.perf_counter_ns() - t0)
        tokens.extend(drafted[:accepted])
        tokens.append(int(r.final_token[0].item()))
        all_acc = accepted == g
        stats.all_accepted_history.append(int(all_acc))
        stats.steps += 1
        stats.total_drafted += g
        stats.total_accepted += accepted
        gamma = gamma_update(gamma, all_acc, min_gamma, max_gamma)
    return tokens[:max_len], stats
