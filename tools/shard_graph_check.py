"""torchrun check of the row-sharded path with graph replay: results of the
captured replays equal the eager first call and the single-GPU xigemm."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, torch.distributed as dist
import paper_2403_06924_b200 as xg
from paper_2403_06924_b200 import sharded
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("nccl")
w, r = dist.get_world_size(), dist.get_rank()
m, k, n = 1024, 2048, 768
a_full = xg.generate("student_t3", m * w, k, 5, 0.0, 1.0)
b = xg.generate("normal", k, n, 6, 0.0, 1.0)
cfg = xg.XigemmConfig(threshold=0.05, scheme=xg.QuantScheme.VectorWise, policy=xg.ReductionPolicy.AvgRule)
a = a_full[r * m:(r + 1) * m].contiguous()
out = torch.empty((m, n), device="cuda")
res = []
for i in range(4):
    a.copy_(a_full[r * m:(r + 1) * m])
    rep = sharded.xigemm_sharded(a, b, cfg=cfg, out=out, rank_rows=[m] * w)
    res.append(out.clone())
ref = xg.xigemm(a_full, b, cfg=cfg).result[r * m:(r + 1) * m]
ok = all(torch.equal(x.view(torch.int32), ref.view(torch.int32)) for x in res)
print(f"rank {r}: graph replays equal single-GPU: {ok}; density {rep.density_a:.4f}", flush=True)
dist.destroy_process_group()
sys.exit(0 if ok else 1)
