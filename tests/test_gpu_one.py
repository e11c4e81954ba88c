"""The one-tile-per-SM dense kernel (attn_one.cu; opt-in with ADASPA_ONE=1) against the
fp64 oracle: the dense, edge-case and rescale parity tests re-run in a fresh interpreter with the
variable set (the library reads it once per process)."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_one_tile_kernel_matches_oracle():
    env = dict(os.environ, ADASPA_ONE="1")
    files = [os.path.join(ROOT, "tests", f) for f in ("test_gpu_parity.py", "test_gpu_edges.py", "test_gpu_rescale.py")]
    r = subprocess.run([sys.executable, "-m", "pytest", *files, "-m", "gpu", "-q", "-p", "no:cacheprovider",
                        "-k", "dense or edge or rescale or end_to_end or hot_path"],
                       env=env, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0 and " passed" in r.stdout, r.stdout[-3000:] + r.stderr[-2000:]
