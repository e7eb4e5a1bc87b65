"""K4b with TMA gather4 record fetches (VGICP_TMA_REC=1, an opt-in kernel: measured 19% slower
than the cp.async cooperative gathers on config 5) stays bit-for-bit
interchangeable: the parity tests of the batched path pass through it (a subprocess, since the
knob is read once per process)."""

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def test_tma_record_gathers_pass_the_batched_parity_tests():
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu",
                        str(ROOT / "tests" / "test_gpu_parity.py"), "-k",
                        "config5_every_factor or config5_blocks or batch_pose_table or "
                        "f32_records or empty_source"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT,
                       env=dict(os.environ, VGICP_TMA_REC="1"))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout
