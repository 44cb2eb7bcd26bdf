"""The reference's C++ API, re-hosted: reference-style call sites compile against
include/prescope_b200.hpp, link libprescope_b200.so and pass (CPU only)."""
import subprocess

from conftest import ROOT


def test_cpp_shim_compiles_and_passes(tmp_path):
    exe = tmp_path / "shim_test"
    lib_dir = ROOT / "paper_2509_23638_b200"
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", str(ROOT / "include"), str(ROOT / "tests/cpp/shim_test.cpp"),
                    "-L", str(lib_dir), "-lprescope_b200", f"-Wl,-rpath,{lib_dir}", "-o", str(exe)], check=True)
    import os
    import shutil
    gold = tmp_path / "ref_trace_desk.tsv"  # the shim writes next to it
    shutil.copy(ROOT / "tests/golden/ref_trace_desk.tsv", gold)
    out = subprocess.run([str(exe)], capture_output=True, text=True,
                         env={**os.environ, "PRESCOPE_GOLDEN_TRACE": str(gold)})
    assert out.returncode == 0, out.stderr
    assert "shim ok" in out.stdout
