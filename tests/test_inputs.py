"""Synthetic input generator (inputs/synth.py): exact gap counts, determinism, structure."""
import numpy as np

from inputs.synth import cloud_mask, heterogeneous_field, make_problem, matern_field, random_mask


def test_random_mask_exact_count_and_determinism():
    m = random_mask(16, 16, 0.5)
    assert (m == 0).sum() == 128
    assert np.array_equal(m, random_mask(16, 16, 0.5))
    assert (random_mask(64, 64, 0.33) == 0).sum() == round(0.33 * 64 * 64)


def test_cloud_mask_is_clustered():
    m = cloud_mask(128, 128, 0.7)
    assert (m == 0).sum() == round(0.7 * 128 * 128)
    # clustered gaps: far more gap-gap neighbours than a random mask of the same density
    same = lambda a: np.mean((a[:, 1:] == 0) & (a[:, :-1] == 0))
    assert same(m) > same(random_mask(128, 128, 0.7)) + 0.1


def test_matern_unit_variance_and_correlation():
    f = matern_field(256, 256, nu=1.5, corr_len=16.0)
    assert abs(f.std() - 1) < 1e-9
    c1 = np.corrcoef(f[:, :-1].ravel(), f[:, 1:].ravel())[0, 1]
    assert c1 > 0.9


def test_heterogeneous_variance_spread():
    z = heterogeneous_field(256)
    q = [z[:128, :128].std(), z[:128, 128:].std(), z[128:, :128].std(), z[128:, 128:].std()]
    assert max(q) / min(q) > 1.5
    assert z.dtype == np.float32


def test_make_problem_hides_gaps():
    truth, z, mask = make_problem(32, 0.5)
    assert np.isnan(z[mask == 0]).all() and np.array_equal(z[mask == 1], truth[mask == 1])
