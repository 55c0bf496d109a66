"""Queue hardening (SURVEY §8c queue pins, §4 layers 3 and 5).

* A unique-tag stress program (tests/queue_stress.cu) drives the product's
  queue primitives (device.cuh) with 10^7 chained tasks through a 256-slot ring
  (~39,000 wrap-arounds), with and without randomized __nanosleep injected
  before pushes and before `processed += n`: every tag is processed exactly
  once, processed == tail == N, and no worker quits while work remains.
* More live tasks than slots must raise ATOS_ERR_QUEUE_OVERFLOW, not hang.
* compute-sanitizer memcheck / racecheck / synccheck over every worker kind of
  the three apps on small graphs (tools/sanitize_run.py)."""
import json
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


@pytest.fixture(scope="module")
def stress_exe(tmp_path_factory):
    exe = tmp_path_factory.mktemp("qs") / "queue_stress"
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-lineinfo",
                           "-o", str(exe), os.path.join(HERE, "queue_stress.cu")])
    return str(exe)


def _run(exe, *args, timeout=180):
    p = subprocess.run([exe, *map(str, args)], capture_output=True, text=True, timeout=timeout)
    return p.returncode, json.loads(p.stdout.strip().splitlines()[-1]) if p.stdout.strip() else None, p.stderr


@pytest.mark.parametrize("fetch,blocks,sleep", [(1, 296, 0), (1, 296, 0x3FF), (32, 148, 0), (32, 592, 0xFF),
                                                (7, 148, 0x1FF), (256, 148, 0)])
def test_unique_tag_stress(stress_exe, fetch, blocks, sleep):
    rc, r, err = _run(stress_exe, 10_000_000, 192, 256, fetch, blocks, hex(sleep))
    assert r is not None, err
    assert rc == 0, r
    assert r["missing"] == 0 and r["duplicated"] == 0 and r["early_exits"] == 0
    assert r["processed"] == r["tail"] == 10_000_000 and r["laps"] >= 39_000


def test_overflow_is_detected_not_hung(stress_exe):
    # a binary tree of 100,000 tags (K = 0) through 256 slots: more live tasks than the ring holds
    rc, r, err = _run(stress_exe, 100_000, 0, 256, 4, 148, 0)
    assert r is not None, err
    assert rc == 1 and r["abort"] == 1  # ABORT_OVERFLOW, reported instead of a hang


SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool", ["memcheck", "synccheck", "racecheck"])
def test_compute_sanitizer(tool):
    """Every app x worker kind x kernel strategy on small graphs under compute-sanitizer."""
    assert os.path.exists(SAN)
    env = dict(os.environ, PYTHONPATH=ROOT)
    p = subprocess.run([SAN, f"--tool={tool}", "--error-exitcode=99", "--print-limit=20", "--target-processes=all",
                        sys.executable, os.path.join(ROOT, "tools", "sanitize_run.py"), tool],
                       capture_output=True, text=True, timeout=1500, env=env)
    tail = (p.stdout + p.stderr)[-4000:]
    assert p.returncode == 0, tail
    assert "ERROR SUMMARY: 0 errors" in p.stdout + p.stderr or "RACECHECK SUMMARY: 0 hazards" in p.stdout + p.stderr, tail
    assert "sanitize_run ok" in p.stdout, tail
