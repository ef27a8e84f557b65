"""The reference's own C++ test suites, compiled UNMODIFIED against the B200
drop-in (include/knng/*.hpp -> include/knng_b200.hpp + libknng_b200.so).

tests/cpp/Makefile `reftests` builds /root/reference/proj/tests/{test_refine,
test_distsim, test_graphopt, test_annsearch, test_evalio, acceptance}.cpp
in place (the sources are read, never copied) with a doctest stand-in
(tests/cpp/shim/doctest.h) into tests/cpp/_bin/.  The GPU box has no
/root/reference, so it runs the binaries built here; where neither the
binaries nor the sources exist the cases skip.

test_distsim exercises the host-side RankWorld only (no GPU): it runs in the
CPU suite.  The others drive the GPU path and are `gpu` tests.
"""
import os
import subprocess
import tempfile

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
BIN = os.path.join(HERE, "cpp", "_bin")


def _binary(name):
    path = os.path.join(BIN, "ref_" + name)
    if not os.path.exists(path):
        subprocess.run(["make", "-s", "-C", os.path.join(HERE, "cpp"), "reftests"],
                       check=False, capture_output=True)
    if not os.path.exists(path):
        pytest.skip("reference suite not built (no /root/reference here)")
    return path


def _run(name, timeout=1200):
    exe = _binary(name)
    with tempfile.TemporaryDirectory() as cwd:  # acceptance writes its GT cache to ./
        res = subprocess.run([exe], capture_output=True, text=True, timeout=timeout, cwd=cwd)
    print(res.stdout[-6000:])
    assert res.returncode == 0, res.stdout[-4000:] + res.stderr[-2000:]
    return res.stdout


def test_reference_distsim_suite():
    out = _run("test_distsim", timeout=300)
    assert "0 failed" in out


@pytest.mark.gpu
@pytest.mark.parametrize("suite", ["test_refine", "test_graphopt", "test_annsearch",
                                   "test_evalio"])
def test_reference_suite_on_b200(suite):
    out = _run(suite)
    assert " 0 failed" in out


@pytest.mark.gpu
def test_reference_acceptance_on_b200():
    out = _run("acceptance", timeout=1800)
    assert "FAIL" not in out
