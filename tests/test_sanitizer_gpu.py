"""compute-sanitizer over every C-ABI entry point (memcheck,
racecheck, synccheck) on C1-sized inputs, plus a positive control: an
undersized output buffer must be reported by memcheck."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _sanitizer():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    exe = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(exe):
        pytest.skip("compute-sanitizer not installed")
    # a pool may replace the tool by a stub that refuses to run (it prints
    # why and exits); then there is nothing to check here -- the earlier clean
    # runs are kept in profiles/r02/sanitize_*.log
    try:
        v = subprocess.run([exe, "--version"], capture_output=True, text=True, timeout=60)
        vout = v.stdout + v.stderr
    except (OSError, subprocess.TimeoutExpired) as e:
        pytest.skip(f"compute-sanitizer not runnable: {e}")
    if v.returncode != 0 or "closed" in vout or "Compute Sanitizer" not in vout:
        pytest.skip("compute-sanitizer unavailable on this host: " + vout.strip()[:200])
    from paper_2512_11473_b200 import build
    build.build()
    return exe


def _run(exe, tool, script, extra=()):
    r = subprocess.run([exe, "--tool", tool, *extra, "--target-processes", "all",
                        "--print-limit", "20", sys.executable, script], cwd=ROOT,
                       capture_output=True, text=True, timeout=900)
    return r.returncode, r.stdout + r.stderr


@pytest.mark.parametrize("tool,extra", [("memcheck", ("--leak-check", "no")), ("racecheck", ()),
                                        ("synccheck", ())])
def test_sanitizer_clean(tool, extra):
    exe = _sanitizer()
    rc, out = _run(exe, tool, "scripts/sanitize_run.py", extra)
    if "closed on this pool" in out:
        pytest.skip(out.strip()[:200])
    assert "sanitize_run ok" in out, out[-3000:]
    if tool == "racecheck":
        assert "RACECHECK SUMMARY: 0 hazards" in out, out[-3000:]
    else:
        assert "ERROR SUMMARY: 0 errors" in out, out[-3000:]
    assert rc == 0


def test_memcheck_catches_undersized_output():
    exe = _sanitizer()
    rc, out = _run(exe, "memcheck", "scripts/sanitize_negative.py", ("--leak-check", "no"))
    if "closed on this pool" in out:
        pytest.skip(out.strip()[:200])
    assert "Invalid __global__ write" in out or "Invalid __global__ write" in out.replace("  ", " "), \
        out[-3000:]
