"""The reference's own unit tests, built unmodified from /root/reference with a
doctest shim (oracle/Makefile target `refcheck`):

* test_grid.cpp against the reference grid.cpp      -> pins the oracle's layer
* test_grid.cpp against the PRODUCT's hb::grid       -> the product passes the
  reference's known-answer tests (16 cases, 1613 assertions)
* test_simnet.cpp against the reference simnet.cpp   -> the fabric the oracle
  executes over behaves as its own tests require
"""
import os
import subprocess

import pytest

from helpers import ROOT

BIN = os.path.join(ROOT, "oracle", "_ref")


@pytest.mark.parametrize("name,cases", [("test_grid_ref", 16), ("test_grid_product", 16), ("test_simnet_ref", 18)])
def test_reference_unit_tests_pass(name, cases):
    exe = os.path.join(BIN, name)
    if not os.path.exists(exe):
        if os.path.isdir("/root/reference/proj"):
            subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "refcheck"], check=True)
        else:
            pytest.skip("reference tests not built and /root/reference absent")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert f"test cases: {cases} | 0 failed" in r.stdout


def test_reference_side_binding_matches_reference():
    """INTEGRATION.md §2's binding (hetsim types -> hetbridge C-ABI), compiled against
    the reference headers, answers every grid/bridge call of a layout sweep exactly
    like the reference grid and the oracle bridge (oracle/refcheck/shim)."""
    exe = os.path.join(BIN, "shim_check")
    if not os.path.exists(exe):
        if os.path.isdir("/root/reference/proj"):
            subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "refcheck"], check=True)
        else:
            pytest.skip("shim check not built and /root/reference absent")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert " 0 mismatches" in r.stdout


@pytest.mark.gpu
def test_reference_side_device_bridge_matches_oracle():
    """The same binding's DeviceBridge (hetsim::grid::BoundaryEdge -> hb_exec_* on
    cuda:0) executed for C1, C2, C3, C3', C5, App-C and a cp
    reduce: forward placement and the backward return equal the oracle's
    bridge_forward / bridge_backward bit for bit (oracle/refcheck/shim/device_check.cpp)."""
    exe = os.path.join(BIN, "shim_device_check")
    if not os.path.exists(exe):
        if os.path.isdir("/root/reference/proj"):
            subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "refcheck"], check=True)
        else:
            pytest.skip("device check not built and /root/reference absent")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " 0 mismatches" in r.stdout
