"""One engine call over several B200s (sym_config.devices): sub-cluster s
runs on devices[s mod D] and the result equals the one-device run bit for
bit -- per-request arrays, batch records with global model/GPU/request ids,
window reductions and the event trace.  Needs >= 2 visible GPUs (gpurun
--gpus 2 / 4); skipped otherwise."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ndev():
    import torch
    return torch.cuda.device_count()


def _c4(dur):
    from paper_2308_07470_b200 import configs
    from paper_2308_07470_b200.workload import generate_arrivals
    sc = configs.c4(dur)
    ticks, midx = generate_arrivals(sc.workload, [m.name for m in sc.models], dur, 42)
    return sc, ticks, midx


def _same(a, b):
    for k in ("req_dispatch", "req_start", "req_finish", "req_batch", "req_outcome",
              "req_arrival", "req_deadline", "req_model"):
        np.testing.assert_array_equal(getattr(a, k), getattr(b, k), err_msg=k)
    for f in ("gpu", "model", "size", "start", "finish", "emitted", "first_index"):
        np.testing.assert_array_equal(a.batches[f], b.batches[f], err_msg=f)
    assert a.drops == b.drops and a.completions == b.completions


@pytest.mark.parametrize("ndev", [2, 4])
def test_multi_device_call_equals_one_device(ndev):
    if _ndev() < ndev:
        pytest.skip(f"needs {ndev} GPUs")
    from paper_2308_07470_b200.simulator import Engine
    sc, ticks, midx = _c4(5.0)
    one = Engine(list(sc.models), sc.gpu_count, sc.policy, shards=sc.shards)
    r1 = one.run_stream(ticks, midx, 5.0)
    w1 = one.window_stats(500_000_000, 4_500_000_000)
    many = Engine(list(sc.models), sc.gpu_count, sc.policy, shards=sc.shards,
                  devices=list(range(ndev)))
    rn = many.run_stream(ticks, midx, 5.0)
    _same(r1, rn)
    assert many.stats["fast_shards"] == 8
    wn = many.window_stats(500_000_000, 4_500_000_000)
    for k in w1:
        np.testing.assert_array_equal(w1[k], wn[k], err_msg=k)
    one.close()
    many.close()


def test_multi_device_policies_and_trace():
    """Overload (eager, the chain) and the event trace across 2 devices."""
    if _ndev() < 2:
        pytest.skip("needs 2 GPUs")
    from paper_2308_07470_b200.scheduler import PolicyConfig
    from paper_2308_07470_b200.simulator import Engine
    sc, ticks, midx = _c4(0.05)
    for pol in (PolicyConfig("eager"), PolicyConfig("timeout", timeout_slo_frac=0.3)):
        kw = dict(shards=sc.shards, record_trace=True)
        a = Engine(list(sc.models), sc.gpu_count, pol, **kw)
        b = Engine(list(sc.models), sc.gpu_count, pol, devices=[0, 1], **kw)
        ra, rb = a.run_stream(ticks, midx, 0.05), b.run_stream(ticks, midx, 0.05)
        _same(ra, rb)
        assert ra.trace == rb.trace
        a.close()
        b.close()


def test_run_scenario_on_all_devices():
    """run_scenario with devices= (the hook every analysis caller uses)."""
    if _ndev() < 2:
        pytest.skip("needs 2 GPUs")
    from paper_2308_07470_b200 import configs, run_scenario
    sc = configs.c4(1.0)
    a = run_scenario(sc)
    b = run_scenario(sc, devices=tuple(range(_ndev())))
    _same(a, b)


def test_unknown_model_reported_in_stream_order():
    if _ndev() < 2:
        pytest.skip("needs 2 GPUs")
    from paper_2308_07470_b200.scheduler import ProtocolError
    from paper_2308_07470_b200.simulator import Engine
    sc, ticks, midx = _c4(0.01)
    midx = midx.copy()
    midx[100] = 5000
    midx[50] = -3
    eng = Engine(list(sc.models), sc.gpu_count, sc.policy, shards=sc.shards, devices=[0, 1])
    with pytest.raises(ProtocolError, match="-3"):
        eng.run_stream(ticks, midx, 0.01)
    eng.close()
