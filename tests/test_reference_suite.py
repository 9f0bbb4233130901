"""The reference's own transfer test suite (proj/tests/transfer_test.cpp,
21 cases incl. 12 randomized end-to-end syncs against its element-level
oracle), compiled unmodified by oracle/Makefile with tests/ref/doctest.h:

* transfer_test_ref    -- linked with the reference's codec.cpp (validates the
                          doctest stand-in; CPU);
* transfer_test_dropin -- linked with paper_2605_06534_b200/shim/codec_shim.cpp
                          instead of codec.cpp, so the reference engine's
                          diff / reslice / apply run on the B200 kernels through
                          the C-ABI (the drop-in proof; GPU);
* transfer_test_dropin_engine -- also engine_shim.cpp instead of engine.cpp:
                          TransferEngine::sync_step itself runs on libwsync's
                          resident-arena engine (GPU).
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_DIR = os.path.join(ROOT, "oracle", "_ref")


def _run(name):
    exe = os.path.join(REF_DIR, name)
    if not os.path.exists(exe):
        pytest.skip(f"{name} not built (needs /root/reference at build time)")
    p = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    return p.returncode, p.stderr


def test_reference_suite_on_reference_codec():
    rc, log = _run("transfer_test_ref")
    assert rc == 0, log[-4000:]
    assert "test cases: 21 | failed: 0" in log


@pytest.mark.gpu
def test_reference_suite_on_b200_kernels():
    rc, log = _run("transfer_test_dropin")
    assert rc == 0, log[-4000:]
    assert "test cases: 21 | failed: 0" in log


@pytest.mark.gpu
def test_reference_suite_on_b200_engine():
    """The sync-level drop-in: engine_shim.cpp replaces engine.cpp (and
    codec_shim.cpp codec.cpp), so every TransferEngine::sync_step of the
    reference's suite -- 8 modes x exactness, the dense fallback, the byte
    accounting of shard-aware and naive pulls, 12 randomized layouts checked
    by the element-level oracle (transfer_cases.hpp) -- runs on libwsync's
    one-GPU engine (ws_plan_create with world 1 hosting every rank)."""
    rc, log = _run("transfer_test_dropin_engine")
    assert rc == 0, log[-4000:]
    assert "test cases: 21 | failed: 0" in log
