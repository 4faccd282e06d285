"""Kernel times of one config under a policy (dev tool):
python tools/policy_ktimes.py C1 60 timeout"""
import sys

sys.path.insert(0, ".")
from paper_2308_07470_b200 import configs  # noqa: E402
from paper_2308_07470_b200.scheduler import PolicyConfig  # noqa: E402
from paper_2308_07470_b200.simulator import Engine  # noqa: E402
from paper_2308_07470_b200.workload import generate_arrivals  # noqa: E402

name, dur, kind = sys.argv[1], float(sys.argv[2]), sys.argv[3]
sc = configs.CONFIGS[name](dur)
ticks, midx = generate_arrivals(sc.workload, [m.name for m in sc.models], dur, 42)
pol = sc.policy if kind == "base" else (PolicyConfig("timeout", timeout_slo_frac=0.3)
                                        if kind == "timeout" else PolicyConfig(kind))
eng = Engine(list(sc.models), sc.gpu_count, pol, shards=sc.shards)
eng.run_stream(ticks, midx, dur)
eng.kernel_times(reset=True)
import torch  # noqa: E402
import numpy as np  # noqa: E402
t = torch.from_numpy(ticks).cuda()
m = torch.from_numpy(midx.astype(np.int32)).cuda()
out, cnt = eng.run_device(t, m, kernel_times=True)
kt = eng.kernel_times()
print(name, kind, len(ticks), {k: round(v, 2) for k, v in cnt.items() if k.startswith("ms_")})
for k, v in sorted(kt.items(), key=lambda kv: -kv[1][1])[:8]:
    print(f"   {k:20s} {v[0]:4d} {v[1]:9.3f} ms")
