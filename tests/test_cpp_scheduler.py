"""The C++ batcher drop-in (include/tangram/scheduler.hpp + latency.hpp,
cost.hpp, rng.hpp, event_log.hpp) against the reference's own scheduler
unit-test expectations (tests/cpp/scheduler_test.cpp restates
proj/tests/scheduler_test.cpp:56-320), and -- where the reference build of
the same test source exists -- byte for byte against the reference headers:
every event of 20 random streams (fire time, trigger, k, slack, patch ids,
placements, free rects) and the whole event log.  The batcher is host code,
so this runs without a GPU; a gpu-marked twin keeps it in the GPU suite."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CPP = os.path.join(ROOT, "tests", "cpp")
REF_INC = "/root/reference/proj/include"


def _run(exe):
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]
    assert out.stdout.rstrip().endswith("scheduler_test: ALL PASS")
    return out.stdout


def check_scheduler_dropin():
    subprocess.check_call(["make", "-s", "-C", CPP, "scheduler_test"])
    ours = _run(os.path.join(CPP, "scheduler_test"))
    assert ours.count("seed ") > 100 and '"event":"invoke"' in ours
    ref_exe = os.path.join(CPP, "scheduler_test_ref")
    if os.path.isdir(REF_INC):  # authoring container: (re)build the reference twin
        subprocess.check_call(["make", "-s", "-C", CPP, "scheduler_test_ref"])
    if os.path.exists(ref_exe):
        assert ours == _run(ref_exe), "drop-in and reference builds differ"


def test_scheduler_dropin_cpp():
    check_scheduler_dropin()


@pytest.mark.gpu
def test_scheduler_dropin_cpp_gpu_suite():
    check_scheduler_dropin()
