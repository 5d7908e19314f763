"""The speculative decode loop on the CUDA backend (SURVEY.md 8(f) f1,
decode.cpp:45-159): transcripts equal the reference's decode on the same toy
model tables, seeds and draw order (SPEC.md:328 transcript equality)."""
import numpy as np
import pytest

from paper_2406_11016_b200.decode import CounterRng, gamma_update


def test_counter_rng_matches_reference_stream(oracle):
    """rng.cpp:12-33: the decode loop's draws are the reference's draws (pinned
    through make_bench_inputs, which reads the same stream at fixed indices)."""
    seed, G, V = 9, 3, 50
    _, _, _, u = oracle.make_bench_batch(seed, 1, G, V)
    rng = CounterRng(seed)
    rng.counter = 2 * (2 * G + 1) * V + G  # bench.cpp:66-73: after the logits and the draft draws
    assert [rng.next_uniform() for _ in range(G + 1)] == list(u[0])


def test_gamma_update():
    assert gamma_update(5, True, 1, 64) == 7 and gamma_update(63, True, 1, 64) == 64
    assert gamma_update(5, False, 1, 64) == 4 and gamma_update(1, False, 1, 64) == 1


@pytest.mark.gpu
@pytest.mark.parametrize("variant", ["exact", "sigmoid"])
@pytest.mark.parametrize("seed,V,div", [(1, 64, 0.5), (2, 1000, 1.0), (3, 257, 0.0), (4, 4099, 2.0)])
def test_decode_transcript_matches_reference(verifier, ref, variant, seed, V, div):
    import torch

    t, d = ref.make_model_pair(seed, V, div)
    t = t.astype(np.float32).astype(np.float64)  # the device holds fp32 tables
    d = d.astype(np.float32).astype(np.float64)
    from paper_2406_11016_b200.decode import decode

    prompt = [seed % V]
    tt = torch.from_numpy(t.astype(np.float32)).cuda()
    dt = torch.from_numpy(d.astype(np.float32)).cuda()
    for dseed in (0, 17):
        ref_tokens, ref_gammas = ref.decode(t, d, prompt, 48, gamma=4, seed=dseed,
                                            backend="reference" if variant == "exact" else "sigmoid")
        tokens, stats = decode(verifier, tt, dt, prompt, 48, gamma=4, seed=dseed, variant=variant)
        assert tokens == ref_tokens.tolist(), f"{variant} seed {seed}/{dseed}: transcript differs"
        assert stats.gamma_history == ref_gammas.tolist()
