"""Oracle pinning: Philox / normal / uniform against vectors produced by the reference's own
proj/src/rng.cpp (tests/golden/make_golden.py), plus the SURVEY.md B.1 literals."""
import json
import os

import numpy as np

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def test_philox_known_answers(oracle):
    for kat in _load("rng_kat.json")["philox"]:
        assert oracle.philox4x32(kat["ctr"], kat["key"]) == kat["out"]
    # Random123 Philox4x32-10 KAT
    assert oracle.philox4x32([0, 0, 0, 0], [0, 0]) == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]


def test_normal_and_uniform_bit_exact_vs_reference(oracle):
    g = _load("rng_kat.json")
    for seed, stream, i, j, hx in g["normal_at"]:
        assert oracle.normal_at(int(seed), stream, i, j) == float.fromhex(hx), (seed, stream, i, j)
    for seed, stream, i, j, hx in g["uniform_at"]:
        assert oracle.uniform_at(int(seed), stream, i, j) == float.fromhex(hx), (seed, stream, i, j)


def test_survey_b1_literals(oracle):
    want = [-0.081874209915891588, -0.68430328303560639, 0.69460481678686981, 1.2962525235399087,
            -0.44270551836996486, -0.16291544953471881]
    got = [oracle.normal_at(0, 1, i, j) for i in range(2) for j in range(3)]
    assert got == want
    assert oracle.normal_at(42, 1, 10, 1999) == 0.7182310716057253
    assert oracle.uniform_at(7, 6, 3, 4) == 0.90953663113359373


def test_gaussian_matrix_block_matches_reference(oracle):
    block = np.array([[float.fromhex(h) for h in row] for row in _load("rng_kat.json")["sketch_block_seed0_11x512"]])
    g = oracle.gaussian_matrix(11, 512, 0, 1)
    assert np.array_equal(g, block)


def test_sparse_sign_pattern_known_answers(oracle):
    for p in _load("sparse_sign_kat.json")["patterns"]:
        rows, signs = oracle.sparse_sign_pattern(p["c"], p["m"], p["seed"], p["zeta"])
        assert rows.tolist() == p["rows"] and signs.tolist() == p["signs"]
        ze = min(p["zeta"], p["c"])
        assert rows.shape == (p["m"], ze)
        for r in rows:  # distinct destinations per column of Omega
            assert len(set(r.tolist())) == ze and r.min() >= 0 and r.max() < p["c"]
        assert set(np.unique(signs).tolist()) <= {-1, 1}


def test_sparse_sign_distribution_is_balanced(oracle):
    rows, signs = oracle.sparse_sign_pattern(22, 20000, 5, 8)
    counts = np.bincount(rows.ravel(), minlength=22)
    assert counts.min() > 0.9 * counts.mean() and counts.max() < 1.1 * counts.mean()
    assert abs(signs.mean()) < 0.02
