"""Compile the reference's OWN test suites unchanged against this repo's
include/roundpipe headers (the drop-in claim), with a Catch2 shim.

/root/reference/proj/tests/{cost_model,partitioner,scheduler,simulator,
transfer_planner,consistency,config_io}_tests.cpp and acceptance.cpp hold the
reference's golden vectors and known-answer tests (frozen 87 slots, 12/108
bubble, protocol makespans 19/21/30 …). They must pass
against our headers exactly as against the reference's. Skipped where the
reference tree is absent (the GPU box).
"""
import os
import shutil
import subprocess
from concurrent.futures import ThreadPoolExecutor

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/proj"
SUITES = ["cost_model", "partitioner", "scheduler", "simulator",
          "transfer_planner", "consistency", "config_io"]

pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference tree absent")


def _build(src, out, include):
    cmd = [shutil.which("g++") or "g++", "-std=c++20", "-O1", f"-I{include}",
           f"-I{ROOT}/tests/catch_shim",
           f'-DROUNDPIPE_CONFIG_DIR="{REF}/configs"',
           '-DROUNDPIPE_CLI_PATH="/nonexistent-cli"', src, "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-4000:]
    return out


@pytest.fixture(scope="module")
def binaries(tmp_path_factory):
    d = tmp_path_factory.mktemp("refsuites")
    jobs = {s: (f"{REF}/tests/{s}_tests.cpp", str(d / s)) for s in SUITES}
    with ThreadPoolExecutor(8) as ex:
        futs = {s: ex.submit(_build, src, out, f"{ROOT}/include")
                for s, (src, out) in jobs.items()}
        futs["acceptance"] = ex.submit(_build, f"{REF}/tests/acceptance.cpp",
                                       str(d / "acceptance"), f"{ROOT}/include")
        return {s: f.result() for s, f in futs.items()}


@pytest.mark.parametrize("suite", SUITES)
def test_reference_unit_suite_passes_on_our_headers(binaries, suite, tmp_path):
    r = subprocess.run([binaries[suite]], capture_output=True, text=True,
                       cwd=tmp_path, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr[-4000:]
    assert "failed: 0" in r.stdout


def test_reference_acceptance_on_our_headers(binaries, tmp_path):
    r = subprocess.run([binaries["acceptance"]], capture_output=True, text=True,
                       cwd=tmp_path, timeout=600)
    lines = [l for l in r.stdout.splitlines() if l.startswith("criterion")]
    assert len(lines) == 10
    # criterion 10 shells out to the reference CLI, which cannot be built
    # here (CLI11 absent) — it fails identically on the reference headers.
    for l in lines[:9]:
        assert "[PASS]" in l, l
