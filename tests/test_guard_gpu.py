"""Guard mode (SYM_GUARD=1): the engine's own memcheck/initcheck, standing in
for compute-sanitizer, which is closed on the GPU pool
(profiles/r02_sanitizer_memcheck.log).  Every device buffer sits between two
4 KiB redzones and every run ends by reading them back (engine.cu
guard_check); the buffer bodies start filled with a poison byte.  The
kernel-family workload (tools/sanitize_case.py, every result against the
oracle) must pass with two different poison bytes -- no write outside a
buffer, and no uninitialised read that changes a result -- and a planted
write one byte past a buffer must be reported by name."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("poison", ["0x00", "0xff", "0x7f"])
def test_kernel_families_clean_under_guard(poison):
    env = dict(os.environ, SYM_GUARD="1", SYM_GUARD_POISON=poison)
    env.pop("SYM_GUARD_SELFTEST", None)
    p = subprocess.run([sys.executable, "tools/sanitize_case.py"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-4000:]
    assert "sanitize workload ok" in p.stdout


def test_guard_reports_a_write_past_a_buffer(monkeypatch):
    from paper_2308_07470_b200 import Engine, PolicyConfig
    from paper_2308_07470_b200.profile import LatencyProfile, ModelSpec
    monkeypatch.setenv("SYM_GUARD", "1")
    monkeypatch.setenv("SYM_GUARD_SELFTEST", "1")
    m = [ModelSpec(0, "m", LatencyProfile.linear(1.0, 5.0, 8), 50_000_000)]
    eng = Engine(m, 2, PolicyConfig("deferred"))
    with pytest.raises(RuntimeError, match="guard: byte 1 past the end of"):
        eng.run_stream(np.array([10, 20], np.int64), np.array([0, 0]), 1.0)
    eng.close()


def test_guard_mode_is_off_by_default(monkeypatch):
    from paper_2308_07470_b200 import Engine, PolicyConfig
    from paper_2308_07470_b200.profile import LatencyProfile, ModelSpec
    monkeypatch.delenv("SYM_GUARD", raising=False)
    monkeypatch.setenv("SYM_GUARD_SELFTEST", "1")  # inert without SYM_GUARD
    m = [ModelSpec(0, "m", LatencyProfile.linear(1.0, 5.0, 8), 50_000_000)]
    eng = Engine(m, 2, PolicyConfig("deferred"))
    res = eng.run_stream(np.array([10, 20], np.int64), np.array([0, 0]), 1.0)
    assert res.n_requests == 2
    eng.close()
