"""bench.py's reference arm (`--impl reference`): the compiled reference's
TransferEngine::sync_step on host cores prints the contract's JSON line with
impl, cpu_baseline and e2e (no GPU needed).  A small model keeps it short."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line():
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref")):
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--model", "qwen2.5-0.5b", "--steps", "1", "--warmup", "1"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    line = json.loads([l for l in p.stdout.splitlines() if l.startswith("{")][-1])
    assert line["impl"] == "reference" and line["unit"] == "GB/s" and line["value"] > 0
    assert line["warmup"] == 1 and line["steps"] == 1
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]


def test_reference_arm_never_maps_libwsync():
    """The reference arm must run the reference alone: the model shapes come
    from manifest.py loaded by path, never through the package (whose
    __init__ maps libwsync.so)."""
    code = ("import sys; sys.argv = ['bench.py']; sys.path.insert(0, %r)\n"
            "import importlib.util\n"
            "spec = importlib.util.spec_from_file_location('bench', %r)\n"
            "b = importlib.util.module_from_spec(spec); spec.loader.exec_module(b)\n"
            "mf = b.load_manifest_module(); assert mf.MODELS['qwen3-8b']()\n"
            "from oracle.oracle import Reference\n"
            "try:\n    Reference()\nexcept OSError:\n    pass\n"
            "print(open('/proc/self/maps').read().count('libwsync'))\n"
            % (ROOT, os.path.join(ROOT, "bench.py")))
    p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300,
                       cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    assert p.stdout.strip().splitlines()[-1] == "0"
