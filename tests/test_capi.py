"""The C-ABI library loads (no GPU needed to load) and exports every symbol include/itercur_b200.h declares."""
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    with open(os.path.join(ROOT, "include", "itercur_b200.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"ITERCUR_API\s+[\w\s\*]+?\b(itercur_\w+)\s*\(", text)))


def test_header_declares_entry_points():
    names = _declared()
    assert "itercur_iterative_cur_device" in names and "itercur_iterative_cur_host" in names
    assert len(names) >= 30


def test_library_builds_loads_and_exports_all_symbols():
    from paper_2509_21963_b200 import _capi, build

    build.build()
    lib = _capi.lib()
    for name in _declared():
        assert hasattr(lib, name), name
    assert sorted(_capi.EXPORTED) == _declared()
    assert lib.itercur_abi_version() == 4


def test_cpu_only_call_fails_loudly_without_device():
    import torch

    if torch.cuda.is_available():
        return
    import numpy as np
    import pytest

    import paper_2509_21963_b200 as E

    with pytest.raises(RuntimeError, match="no CUDA device"):
        E.iterative_cur(np.eye(4), b=2)


def test_host_helpers_without_device():
    import paper_2509_21963_b200 as E

    assert [E.sketch_rows_for_block(b) for b in (1, 10, 50)] == [1, 11, 55]
    assert abs(E.adjusted_threshold(1.0, 0.0, 1e-10, 100) - 1 / 4.98) < 5e-4 / 4.98
