"""MinRule density against M at C3 under PerTensor (Student-t(3)): the statistic
min|D_F| is 0 in every row and column, so every entry is kept at any M."""
import sys, os
sys.path.insert(0, '/root/repo')
import paper_2403_06924_b200 as xg
a = xg.generate("student_t3", 8192, 8192, 1)
b = xg.generate("student_t3", 8192, 8192, 2)
for M in [1e-3, 1, 10, 100, 1e3, 1e4, 3e4, 1e5, 1e6, 1e7]:
    r = xg.xigemm(a, b, cfg=xg.XigemmConfig(threshold=M, scheme=xg.QuantScheme.PerTensor, policy=xg.ReductionPolicy.MinRule))
    print(M, r.density_a, r.density_b, int(r.path), r.nnz_a, r.nnz_b)
