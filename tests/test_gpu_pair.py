"""The CTA-pair kernel (attn_pair.cu, cta_group::2; opt-in with ADASPA_PAIR=1) against
the fp64 oracle.  The library reads ADASPA_PAIR once per process, so each case runs in a fresh
interpreter (tests/pair_check.py) with the variable set."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("case", ["dense", "sparse"])
def test_pair_kernel_matches_oracle(case):
    env = dict(os.environ, ADASPA_PAIR="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "pair_check.py"), case],
                       env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "pair ok" in r.stdout


def test_pair_kernel_rescale_path():
    """The pair kernel's O-rescale path (pv_done barriers) on the ramped-logit workload of
    tests/test_gpu_rescale.py (d = 128, block 128: the shapes the pair kernel serves)."""
    env = dict(os.environ, ADASPA_PAIR="1")
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(ROOT, "tests", "test_gpu_rescale.py"),
                        "-m", "gpu", "-q", "-p", "no:cacheprovider", "-k", "128-128"],
                       env=env, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0 and "1 passed" in r.stdout, r.stdout[-3000:] + r.stderr[-2000:]
