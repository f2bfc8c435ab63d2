"""Host logic of the experiment harness (proj/src/bench.cpp restated in benchtool.py): source
parsing and its error texts, and the CSV layout / row order, with the engine calls replaced by
recording fakes (no device needed)."""
import pytest

from paper_2509_21963_b200 import benchtool as B


@pytest.mark.parametrize("src,msg", [
    ("file.mtx", "matrix source must start with 'gen:' or 'mm:'"),
    ("gen:lowrank", "generator spec 'gen:lowrank' needs arguments"),
    ("gen:lowrank:10,5", "wrong number of generator arguments in 'gen:lowrank:10,5'"),
    ("gen:lowrank:10,x,3", "bad generator argument 'x' in 'gen:lowrank:10,x,3'"),
    ("gen:lowrank:10,5 ,3", "bad generator argument '5 ' in 'gen:lowrank:10,5 ,3'"),
    ("gen:lowrankpd:10,5", "wrong number of generator arguments in 'gen:lowrankpd:10,5'"),
    ("gen:lehmer:3,4", "wrong number of generator arguments in 'gen:lehmer:3,4'"),
    ("gen:expdecay:10", "wrong number of generator arguments in 'gen:expdecay:10'"),
    ("gen:bogus:3", "unknown generator kind 'bogus'"),
    ("gen:lowrank:10,5,6", "generator rank must lie in [1, min(m, n)]"),
    ("gen:lowrank:0,5,1", "generator dimensions must be positive"),
    ("gen:expdecay:10,1.5", "singular-value ratio must lie in (0, 1)"),
    ("gen:lowrankpd:10,5,2,1.0", "diagonal decay must lie in (0, 1)"),
])
def test_load_matrix_errors(src, msg):
    # every case fails before any device work (the reference validates in the same order)
    with pytest.raises(ValueError) as e:
        B.load_matrix(src, 0, device="cpu")
    assert str(e.value) == msg


def test_getline_tokenisation_and_stod():
    assert B._tokens("1,2,") == ["1", "2"]  # std::getline drops the trailing empty token
    assert B._tokens(",1") == ["", "1"]
    assert B._parse_index_args(" 7,+3", 2, 2, "s") == [7, 3]
    assert B._stod("0.25abc") == 0.25  # std::stod parses the longest prefix
    with pytest.raises(ValueError):
        B._stod("abc")


def test_lehmer_and_lowrank_pd_on_cpu_tensors():
    import numpy as np

    a = B.testmat.lehmer(4, device="cpu").numpy()
    i = np.arange(4)
    assert np.array_equal(a, (np.minimum.outer(i, i) + 1.0) / (np.maximum.outer(i, i) + 1.0))


class _F:
    def __init__(self, rank):
        self.rank = rank
        self._run = None


class _T:
    final_rho = 0.125


def test_threshold_csv_layout(monkeypatch):
    calls = []
    monkeypatch.setattr(B, "load_matrix", lambda src, seed: ("A", src, seed))
    monkeypatch.setattr(B, "iterative_cur", lambda a, **kw: (calls.append(("it", kw["seed"])) or (_F(7), _T())))
    monkeypatch.setattr(B, "slupp_cur", lambda a, r, seed: (calls.append(("sl", r, seed)) or _F(r)))
    monkeypatch.setattr(B, "true_relative_error", lambda a, f: 0.1)
    monkeypatch.setattr(B, "sketched_relative_error", lambda a, f, b, seed: 1.0 / 3.0)
    cfg = B.ExperimentConfig(matrix_source="gen:lehmer:5", b=4, reps=2, seed_base=10)
    csv = B.run_threshold(cfg)
    lines = csv.splitlines()
    assert lines[0] == "method,rep,final_rank,rel_error_true,rel_error_sketched,wall_time_s"
    assert [ln.split(",")[:3] for ln in lines[1:]] == [["IterativeCUR", "0", "7"], ["IterativeCUR", "1", "7"],
                                                       ["s-LUPP", "0", "7"], ["s-LUPP", "1", "7"]]
    assert lines[1].split(",")[3:5] == ["0.10000000000000001", "0.125"]
    assert lines[3].split(",")[4] == "0.33333333333333331"  # %.17g
    assert len(lines[1].split(",")[5].split(".")[1]) == 6  # %.6f
    assert calls == [("it", 10), ("sl", 7, 10), ("it", 11), ("sl", 7, 11)]


def test_common_validation():
    with pytest.raises(ValueError, match="repetitions must be at least 1"):
        B.run_threshold(B.ExperimentConfig(matrix_source="gen:lehmer:3", reps=0))

    class H:
        rows, cols = 5, 4

    for ranks, msg in [([], "rank list must not be empty"), ([3, 2], "rank list must be sorted ascending"),
                       ([0], "ranks must be positive"), ([5], "rank 5 exceeds min(m, n) = 4")]:
        with pytest.raises(ValueError, match=msg.replace("(", r"\(").replace(")", r"\)")):
            B._validate_ranks(B.ExperimentConfig(ranks=ranks), H())


def test_cli_reports_errors(capsys):
    rc = B.main(["threshold", "--matrix", "nope", "--out", "/tmp/_itercur_never_written.csv"])
    assert rc == 1
    assert "error: matrix source must start with 'gen:' or 'mm:'" in capsys.readouterr().err
