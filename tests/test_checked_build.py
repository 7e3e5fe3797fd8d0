"""The GPU suite against the CHECKED build of libcdr (-DCDR_CHECKED:
device-side bounds checks on texel indices, hit-cache triangle ids, candidate
list indices, boundary segment picks, radix-sort scatter positions; traversal
stack bounds trap in every build). compute-sanitizer is closed on the GPU pool
(it left GPUs needing a reset), so this is the memory-safety run: every parity
test re-runs with the checks on and must pass; a violated check traps and
fails its call with a CUDA error."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_2103_15208_b200", "lib", "checked", "libcdr.so")

pytestmark = pytest.mark.gpu


def _env():
    if not os.path.exists(CHECKED):
        pytest.fail(f"{CHECKED} missing: __graft_entry__.build() builds it")
    return dict(os.environ, CDR_LIB=CHECKED)


def test_checked_library_is_the_checked_build():
    code = ("from paper_2103_15208_b200 import api; L = api.load_library(); "
            "print(api.LIB_PATH, L.cdr_build_flags())")
    r = subprocess.run([sys.executable, "-c", code], env=_env(), cwd=ROOT, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr
    path, flags = r.stdout.split()
    assert path == CHECKED and int(flags) & 1


def test_gpu_suite_under_bounds_checks():
    r = subprocess.run([sys.executable, "-m", "pytest", "tests", "-m", "gpu", "-q", "-x", "-p", "no:cacheprovider",
                        "--ignore", "tests/test_checked_build.py", "--ignore", "tests/test_integration.py"],
                       env=_env(), cwd=ROOT, capture_output=True, text=True, timeout=1800)
    tail = r.stdout[-3000:] + r.stderr[-2000:]
    assert r.returncode == 0, tail
    assert "CDR_DCHECK failed" not in r.stdout + r.stderr, tail
