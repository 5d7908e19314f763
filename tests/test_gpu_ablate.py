"""Scale ablation on the CUDA backend (ablate.cpp:42-103):
every transcript of tools/ablate.py -- the exact baseline and the sigmoid
variant at each bound magnitude, full precision and the binary16 emulation --
equals the compiled reference's decode on the same fp32-rounded toy tables
(exact: Backend::fused, as ablate.cpp:51-57 scores against; sigmoid:
Backend::sigmoid with emulate_half), so the report rows (acceptance,
normalized edit distance) are the reference's."""
import numpy as np
import pytest

from tests.parity import log_parity

pytestmark = pytest.mark.gpu


def test_normalized_edit_distance():
    from tools.ablate import normalized_edit_distance as ned

    assert ned([], []) == 0.0
    assert ned([1, 2, 3], [1, 2, 3]) == 0.0
    assert ned([1, 2, 3], [1, 3]) == pytest.approx(1 / 3)
    assert ned([1, 2], [3, 4, 5, 6]) == 1.0


@pytest.mark.parametrize("profile", ["asr", "text"])
def test_ablation_transcripts_match_reference(verifier, ref, profile):
    from tools.ablate import ablate_scale, tables

    seeds, mags, max_len = (1, 2), (1e1, 1e3, 1e5), 64
    got = {}
    rows = ablate_scale(verifier, profile, mags, seeds, max_len, transcripts=got)
    n = 0
    for (seed, m, half), toks in got.items():
        t, d = (x.astype(np.float64) for x in tables(seed, profile))
        if m is None:
            want, _ = ref.decode(t, d, [0], max_len, gamma=5, seed=seed, backend="fused")
        else:
            want, _ = ref.decode(t, d, [0], max_len, gamma=5, seed=seed, backend="sigmoid", alpha=-m, beta=m,
                                 emulate_half=half)
        assert toks == want.tolist(), f"{profile} seed {seed} m={m} half={half}: transcript differs"
        n += 1
    for r in rows:
        log_parity(f"ablation {profile} +-{r['beta']:g} {r['precision']}: accept {r['accept_rate_mean']:.3f} "
                   f"divergence {r['divergence_mean']:.3f}", len(seeds), 0)
    assert n == len(seeds) * (1 + 2 * len(mags))
