import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from synth import LayoutConfig
from tests import harness
from paper_2505_24034_b200 import runner
mc, sdt, ddt = int(sys.argv[1]), sys.argv[2], sys.argv[3]
cfg = LayoutConfig("t", "toy", 3, 2, 4, sdt, ddt, "colocated")
job = runner.SyncJob(runner.JobSpec(cfg, 1), fill=False)
job.plan.set_max_ctas(0, mc)
info = job.plan.device_info(0)
print("items", info.n_cast_items, info.n_fp8_items, info.n_fp8_pull_items, flush=True)
ol = oracle.Layout(job.model, 3, 2, 4, sdt, ddt)
src = harness.host_src(ol, 1)
for r, t in job.src.items():
    t.copy_(torch.from_numpy(src[r]))
for t in job.dst.values():
    t.fill_(0)
torch.cuda.synchronize()
t0 = time.time()
job.sync()
torch.cuda.synchronize()
print("sync done", time.time() - t0, flush=True)
want = harness.oracle_dst(ol, src, 0)
ok = all(np.array_equal(t.cpu().numpy(), want[g]) for g, t in job.dst.items())
print("parity", ok, flush=True)
