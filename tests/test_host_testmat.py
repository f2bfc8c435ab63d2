"""oracle/host_testmat.py: the reference arm's host-side BASELINE generators (no engine library)."""
import numpy as np

from oracle import host_testmat as H


def test_configs_match_the_engine_table():
    from paper_2509_21963_b200 import testmat

    assert H.CONFIGS == testmat.CONFIGS


def test_rbf_entries_follow_the_recipe(oracle):
    a = H.generate(3, 40, 30)
    i, j = 7, 11
    x = [oracle.uniform_at(1, 4, i, d) for d in range(3)]
    y = [oracle.uniform_at(1, 5, j, d) for d in range(3)]
    want = np.exp(-sum((p - q) ** 2 for p, q in zip(x, y)) / (2 * 0.25))
    assert a.flags.f_contiguous and abs(a[i, j] - want) <= 1e-15


def test_low_rank_plus_noise_spectrum(oracle):
    a = H.generate(4, 1200, 900)
    s = np.linalg.svd(a, compute_uv=False)
    # 400 signal directions with sigma_k = 0.97^k, then the 1e-10 noise floor
    assert s[399] > 1e-7 and s[401] < 1e-7
    assert abs(a[3, 5] - (a[3, 5] - 1e-10 * oracle.normal_at(1, 6, 3, 5))) < 2e-9


def test_orthogonal_configs_have_the_stated_singular_values():
    a = H.generate(1, 120, 120)
    s = np.linalg.svd(a, compute_uv=False)
    assert np.allclose(s, 10.0 ** (-np.arange(120) / 20.0), rtol=1e-9, atol=1e-15)
