"""The reference-side binding of INTEGRATION.md §1 (examples/reference_shim.cpp):
built against the reference's own headers and compiled library, it prices with
the reference's run() and, through the C-ABI, with the B200 library."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "examples", "_bin", "reference_shim")


def test_reference_shim_builds():
    if not os.path.exists("/root/reference/proj/core/include/hjmsv/solver.hpp"):
        pytest.skip("reference headers absent (the GPU box runs the prebuilt binary)")
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "examples")], check=True)
    assert os.path.exists(BIN)


@pytest.mark.gpu
def test_reference_shim_matches_reference_run(gpu):
    if not os.path.exists(BIN):
        pytest.skip("examples/_bin/reference_shim not built")
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    rows = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert {(r["case"], r["mode"]) for r in rows} == {
        (c, m) for c in ("zcb", "caplet", "caplet_timefn") for m in ("strict", "fast")}
    for r in rows:
        assert r["grid_rel"] <= 1e-10 and r["price_rel"] <= 1e-10, r


CDEMO = os.path.join(ROOT, "examples", "_bin", "capi_demo")


def test_capi_from_plain_c():
    """include/hjmsv_b200.h compiles as C11 (-pedantic) and the host helpers run."""
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "examples"), CDEMO], check=True)
    out = subprocess.run([CDEMO], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert json.loads(out.stdout.splitlines()[0])["abi"] >= 1


@pytest.mark.gpu
def test_capi_from_plain_c_solves(gpu):
    if not os.path.exists(CDEMO):
        pytest.skip("examples/_bin/capi_demo not built")
    out = subprocess.run([CDEMO], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "zcb_price" in out.stdout
