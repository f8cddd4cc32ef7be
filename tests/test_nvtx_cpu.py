"""NVTX stage ranges: with EMM_NVTX=1 the hot path's stage entry
points are wrapped in named ranges; without it they are the plain functions."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PROBE = """
import paper_2507_10069_b200.ops as ops
from paper_2507_10069_b200.pipeline import HotPath
from paper_2507_10069_b200.decode import DecodeSession
print(int(ops.NVTX), int(hasattr(HotPath.encode, '__wrapped__')),
      int(hasattr(HotPath.prefill, '__wrapped__')), int(hasattr(DecodeSession.step, '__wrapped__')))
"""


def _run(env_val):
    env = dict(os.environ, EMM_NVTX=env_val)
    out = subprocess.run([sys.executable, "-c", PROBE], cwd=ROOT, env=env, capture_output=True,
                         text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    return out.stdout.split()


def test_nvtx_ranges_on_and_off():
    assert _run("1") == ["1", "1", "1", "1"]
    assert _run("") == ["0", "0", "0", "0"]
