"""Time the Python REFERENCE (batchsym, /root/reference) on this host: its
run_stream on the bench workload's C4 sub-cluster 0 (6 s of the trace) and
its own scale-bench with one worker (dev tool; build container only -- the
reference does not travel to the GPU box)."""
import sys, time, os
sys.path.insert(0, '/root/reference/pkg/src')
sys.path.insert(0, '/root/repo')
from batchsym.simulator import Engine as REngine
from batchsym import scalebench as RSB
from paper_2308_07470_b200 import configs
from paper_2308_07470_b200.workload import generate_arrivals
dur = 6.0
sc = configs.c4(dur)
ticks, midx = generate_arrivals(sc.workload, [m.name for m in sc.models], dur, configs.SEED)
ms, gpus, ids = configs.shard_scenarios(sc)[0]
sel = (midx >= ids[0]) & (midx <= ids[-1])
t, m = ticks[sel], midx[sel] - ids[0]
import batchsym.profile as RP, batchsym.scheduler as RS
rmodels = [RP.ModelSpec(x.model_id, x.name, RP.LatencyProfile(x.profile.kind, x.profile.max_batch, x.profile.alpha_ns, x.profile.beta_ns, x.profile.lat_ns), x.slo_ns) for x in ms]
eng = REngine(rmodels, gpus, RS.PolicyConfig("deferred"))
t0 = time.time(); res = eng.run_stream(t, m, dur); el = time.time() - t0
print(f"reference run_stream C4 sub-cluster 0, {dur:g} s trace: {len(t)} requests in {el:.2f} s = {len(t)/el:.0f} req/s (1 core)")
p = RSB.bench_workers(1, 64, 128, 5.0)
print(f"reference scale-bench workers=1 (64 models, 128 GPUs): {p.throughput_rps:.0f} decisions/s")
print("cpu", os.cpu_count())
