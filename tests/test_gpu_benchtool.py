"""GPU checks of the experiment-harness pieces: the reference generator kinds against numpy
restatements on the oracle's (reference-pinned) Philox normals, the sketched residual of
finished factors (make_sketch + downdate_col_residual, sketch.cpp:10-41) against the oracle's
sketch, and a threshold run end to end."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_generators_match_numpy(engine, oracle):
    from paper_2509_21963_b200 import testmat

    m, n, r, seed = 300, 200, 12, 5
    left = oracle.gaussian_matrix(m, r, seed, stream=testmat.GEN_LEFT)
    right = oracle.gaussian_matrix(n, r, seed, stream=testmat.GEN_RIGHT)
    ref = left @ right.T
    got = testmat.low_rank(m, n, r, seed).cpu().numpy()
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()
    pd = testmat.low_rank_pd(m, n, r, 0.0, seed).cpu().numpy()
    d = min(m, n)
    ratio = 1e-12 ** (1.0 / (d - 1))
    diag = np.cumprod(np.r_[1.0, np.full(d - 1, ratio)])
    assert np.abs(np.diag(pd - got) - diag).max() <= 1e-12
    ed = testmat.exp_decay(64, 0.5, seed).cpu().numpy()
    s = np.linalg.svd(ed, compute_uv=False)
    assert np.allclose(s, 0.5 ** np.arange(64), rtol=1e-10, atol=1e-14)


def test_sketched_residual_matches_oracle(engine, oracle):
    rng = np.random.default_rng(3)
    a = oracle.random_gaussian(400, 30, 1) @ oracle.random_gaussian(300, 30, 2).T + 1e-6 * rng.standard_normal((400, 300))
    b, seed = 8, 4
    f, t = engine.iterative_cur(a, epsilon=1e-3, b=b, seed=seed)
    # the run's own estimator reproduces its final rho (a residual of ||GA||-sized terms:
    # rounding is absolute in units of rho = 1)
    rho = engine.sketched_relative_error(a, f, b, seed)
    assert abs(rho - t.final_rho) <= 1e-12
    # another estimator and the s-LUPP baseline, against numpy on the oracle's sketch
    base = engine.slupp_cur(a, 20, seed=7)
    got = engine.sketched_relative_error(a, base, 12, 9)
    y, ga, _ = oracle.sketch(a, 12, 9)
    I, J = base.row_indices, base.col_indices
    x = a[np.ix_(I, J)]
    ref = np.linalg.norm(y - y[:, J] @ np.linalg.solve(x, a[I, :])) / np.linalg.norm(y)
    assert abs(got - ref) <= 1e-12 + 1e-8 * ref
    with pytest.raises(ValueError, match="block exceeds row count"):
        engine.sketched_relative_error(a, base, 401, 0)


def test_threshold_run(engine, tmp_path):
    from paper_2509_21963_b200 import benchtool

    out = tmp_path / "t.csv"
    rc = benchtool.main(["threshold", "--matrix", "gen:lowrankpd:600,400,30", "--b", "10", "--eps", "1e-6",
                         "--reps", "2", "--seed", "3", "--out", str(out)])
    assert rc == 0
    rows = [ln.split(",") for ln in out.read_text().splitlines()]
    assert rows[0] == ["method", "rep", "final_rank", "rel_error_true", "rel_error_sketched", "wall_time_s"]
    assert [r[0] for r in rows[1:]] == ["IterativeCUR", "IterativeCUR", "s-LUPP", "s-LUPP"]
    for r in rows[1:]:
        assert int(r[2]) > 0 and float(r[3]) < 1e-3 and float(r[4]) < 1e-3
    # fixed-rank and block-size sweeps run through the same engine calls
    csv = benchtool.run_fixed_rank(benchtool.ExperimentConfig(matrix_source="gen:lehmer:200", b=8, ranks=[16, 32]))
    lines = csv.splitlines()
    assert lines[0] == "method,rank,rep,rel_error,wall_time_s" and len(lines) == 7
    assert [ln.split(",")[0] for ln in lines[1:]] == ["IterativeCUR"] * 2 + ["TSVD"] * 2 + ["s-LUPP"] * 2
    assert lines[4].startswith("TSVD,32,0,")
