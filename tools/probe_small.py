import sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2308_07470_b200 import load_scenario
from paper_2308_07470_b200.simulator import Engine
from paper_2308_07470_b200.workload import generate_arrivals
for name in ("table2_resnet50", "table2_inceptionresnet", "fig2_flattop"):
    sc = load_scenario(name)
    t, m = generate_arrivals(sc.workload, [x.name for x in sc.models], sc.duration_s, sc.seed)
    eng = Engine(list(sc.models), sc.gpu_count, sc.policy)
    eng.run_stream(t, m, sc.duration_s)
    eng.kernel_times(reset=True)
    td = torch.from_numpy(t).cuda(); md = torch.from_numpy(m.astype(np.int32)).cuda()
    out, cnt = eng.run_device(td, md, kernel_times=True)
    kt = eng.kernel_times()
    print(name, len(t), {k: (round(v, 3) if isinstance(v, float) else v) for k, v in cnt.items() if k in ("fast_shards", "fast_fail_mask", "ms_total", "ms_fast", "ms_chain", "ms_fresh")})
    for k, v in sorted(kt.items(), key=lambda kv: -kv[1][1])[:4]:
        print("   ", k, v[0], round(v[1], 3))
