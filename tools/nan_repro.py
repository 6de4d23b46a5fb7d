import sys; sys.path.insert(0, "/root/repo")
import torch, paper_2403_06924_b200 as xg
from paper_2403_06924_b200 import sharded
a = torch.zeros((3, 8), device="cuda"); b = torch.zeros((8, 4), device="cuda")
a[1, 2] = float("nan")
for g in (1, 2):
    try:
        sharded.xigemm_sharded_local(a, b, nranks=g)
    except Exception as e:
        print(g, type(e).__name__, e)
try:
    xg.xigemm(a, b)
except Exception as e:
    print("single", type(e).__name__, e)
