"""The reference's own optimizer tests (proj/tests/test_optim.cpp), ported 1:1 onto
the header-only C++ shim (include/minicollie_b200/optim.hpp) and run on the GPU:
reference-shaped host code dropping in on libmco."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_2312_00407_b200", "_build", "test_shim")


@pytest.mark.gpu
def test_reference_optim_tests_through_cpp_shim():
    if not os.path.exists(BIN):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


def test_shim_header_compiles_without_gpu(tmp_path):
    src = tmp_path / "t.cpp"
    src.write_text('#include "minicollie_b200/optim.hpp"\n'
                   'int main(){ return minicollie::optim::is_fused('
                   'minicollie::optim::Kind::kLomo) ? 0 : 1; }\n')
    lib = os.path.join(ROOT, "paper_2312_00407_b200", "_build")
    subprocess.run(["g++", "-std=c++20", "-I", os.path.join(ROOT, "include"), str(src), "-o",
                    str(tmp_path / "t"), "-L", lib, "-lmco", f"-Wl,-rpath,{lib}"], check=True)
    assert subprocess.run([str(tmp_path / "t")]).returncode == 0
