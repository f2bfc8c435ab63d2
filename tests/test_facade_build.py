"""The C++ facade (include/itercur/driver_b200.hpp) builds with g++, links the C-ABI library and
exports the reference's C++ entry points (itercur::iterative_cur & co.); no GPU needed."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_facade_builds_and_exports_reference_api():
    from paper_2509_21963_b200 import build

    build.build()
    lib = build.build_facade()
    out = subprocess.run(["nm", "-DC", "--defined-only", lib], capture_output=True, text=True, check=True).stdout
    for sym in ["itercur::iterative_cur(itercur::MatrixHandle const&, itercur::StoppingConfig const&, "
                "itercur::SelectionMethod const&, itercur::SelectionMethod const&, unsigned long, "
                "std::function<void (itercur::CurFactors const&, itercur::IterationRecord const&)> const&)",
                "itercur::true_relative_error(itercur::MatrixHandle const&, itercur::CurFactors const&)",
                "itercur::slupp_cur(itercur::MatrixHandle const&, long, unsigned long)",
                "itercur::FactoredPinv::solve(itercur::DenseMatrix const&) const",
                "itercur::adjusted_threshold(double, double, double, long)"]:
        assert sym in out, sym
    # the facade only maps types: it carries no CUDA code of its own and links the engine
    ldd = subprocess.run(["ldd", lib], capture_output=True, text=True).stdout
    assert "libitercur_b200.so" in ldd


def test_native_facade_test_compiles():
    from paper_2509_21963_b200 import build

    build.build()
    exe = os.path.join(ROOT, "tests", "native", "test_facade")
    compile_facade_test(exe)
    assert os.path.exists(exe)


def compile_facade_test(exe):
    from oracle import oracle

    oracle.build()
    pkg = os.path.join(ROOT, "paper_2509_21963_b200")
    odir = os.path.join(ROOT, "oracle")
    cmd = ["g++", "-O2", "-std=c++17", "-I" + os.path.join(ROOT, "include"), "-I" + odir,
           os.path.join(ROOT, "tests", "native", "test_facade.cpp"), "-L" + pkg, "-litercur_facade", "-litercur_b200",
           "-L" + odir, "-loracle", f"-Wl,-rpath,{pkg}", f"-Wl,-rpath,{odir}", "-o", exe]
    subprocess.run(cmd, check=True)
