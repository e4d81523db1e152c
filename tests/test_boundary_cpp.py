"""Runs the C++ drop-in test (tests/cpp/test_boundary.cpp, prebuilt by
__graft_entry__.build() against the reference's own types and sources) on the
GPU: build_operator / apply_operator / b_inner / arnoldi_run / ritz_extract /
krylov_schur_restart / solve_quadratic with the SPEC signatures, CostLedger
charges, SPEC's hand examples and error categories."""
import json
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

EXE = os.path.join(ROOT, "tests", "cpp", "_build", "test_boundary")


def test_cxx_dropin_runs():
    if not os.path.exists(EXE):
        pytest.skip("tests/cpp/_build/test_boundary not built (needs /root/reference at build time)")
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["checks"] >= 30
    led = out["solve_ledger_json"]
    assert led["fa"]["ops"] == 1 and led["fb"]["ops"] > 0 and led["flops_per_mac"] == 2.0
