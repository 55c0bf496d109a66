"""Queue hardening (SURVEY §8c queue pins, §4 layers 3 and 5).

* A unique-tag stress program (tests/queue_stress.cu) drives the product's
  queue primitives (device.cuh) with 10^7 chained tasks through a 256-slot ring
  (~39,000 wrap-arounds), with and without randomized __nanosleep injected
  before pushes and before `processed += n`: every tag is processed exactly
  once, processed == tail == N, no worker quits while work remains, and a
  message-passing litmus holds (a consumer always sees the payload the
  producer wrote with the atomic whose result decided the push).
* More live tasks than slots must raise ATOS_ERR_QUEUE_OVERFLOW, not hang.
* A bounds-checked build of the library (-DATOS_CHECKED, device.cuh ATOS_CHK)
  over every worker kind of the three apps on small graphs
  (tools/sanitize_run.py), and a malformed graph that must trip a check.
  (compute-sanitizer is closed on this pool: its runs left GPUs needing a
  reset, so it is not invoked.)"""
import json
import os
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
    assert r["mp_violations"] == 0  # relaxed slot publication after a returning atomic
    assert r["processed"] == r["tail"] == 10_000_000 and r["laps"] >= 39_000


def test_overflow_is_detected_not_hung(stress_exe):
    # a binary tree of 100,000 tags (K = 0) through 256 slots: more live tasks than the ring holds
    rc, r, err = _run(stress_exe, 100_000, 0, 256, 4, 148, 0)
    assert r is not None, err
    assert rc == 1 and r["abort"] == 1  # ABORT_OVERFLOW, reported instead of a hang


@pytest.fixture(scope="module")
def checked_lib(tmp_path_factory):
    """libatos built with -DATOS_CHECKED: every index derived from device data
    (popped task words, CSR offsets, column entries) is bounds-checked on the
    device; a failure is reported as ATOS_ERR_CUDA naming file:line.  (This is
    the out-of-bounds detector: compute-sanitizer is closed on this pool.)"""
    sys.path.insert(0, ROOT)
    from paper_2112_00132_b200 import build as b
    out = str(tmp_path_factory.mktemp("chk") / "libatos_checked.so")
    subprocess.check_call([b.nvcc(), *b.NVCC_FLAGS, "-DATOS_CHECKED", "-I", os.path.join(ROOT, "include"), "-o", out,
                           *b.sources(), "-ldl"])
    return out


def test_bounds_checked_build(checked_lib):
    """Every app x worker kind x kernel strategy on small graphs with the
    bounds-checked library (tools/sanitize_run.py): no check fires and the
    results pass their invariants."""
    env = dict(os.environ, PYTHONPATH=ROOT, ATOS_LIB=checked_lib)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_run.py"), "memcheck"],
                       capture_output=True, text=True, timeout=1200, env=env)
    tail = (p.stdout + p.stderr)[-4000:]
    assert p.returncode == 0, tail
    assert "sanitize_run ok" in p.stdout, tail


def test_bounds_check_fires(checked_lib):
    """The checks are live: a graph whose column names vertex 7 of 3 (created
    without ATOS_GRAPH_VALIDATE, so the library trusts it) is caught at graph
    create, as an error naming the check instead of an out-of-bounds access."""
    code = ("import numpy as np, paper_2112_00132_b200 as atos\n"
            "try:\n"
            "    atos.Graph(np.array([0, 1, 2, 2], np.int64), np.array([1, 7], np.int32))\n"
            "    print('no error')\n"
            "except atos.AtosError as e:\n"
            "    print('caught', e.name, e)\n")
    env = dict(os.environ, PYTHONPATH=ROOT, ATOS_LIB=checked_lib)
    p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, env=env)
    assert "caught CUDA" in p.stdout and "bounds check failed at kernels.cuh" in p.stdout, p.stdout + p.stderr
