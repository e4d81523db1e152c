"""Host m x m kernels of the Krylov-Schur driver (csrc/host/dense.cpp): Schur
form, reordering, real basis of an invariant subspace (compiled C++ unit test)."""
import os
import subprocess

from conftest import ROOT


def test_dense_kernels(tmp_path):
    exe = tmp_path / "test_dense"
    r = subprocess.run(["g++", "-O2", "-std=c++17", "-o", str(exe),
                        os.path.join(ROOT, "tests", "cpp", "test_dense.cpp"),
                        os.path.join(ROOT, "paper_2112_14064_b200", "csrc", "host", "dense.cpp")],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout
    assert r.stdout.count(" ok") == 7  # 5 random + 2 degenerate-cluster matrices
    assert r.stdout.count("zok") == 5  # complex_schur_c on random complex matrices
    assert r.stdout.count(" rok") == 7  # real_schur_reorder on the same 7 matrices
