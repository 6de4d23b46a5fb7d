# One-box check of bench.py's --gpus N > 1 path (row-sharded, weak scaling):
# two ranks on one GPU over gloo (eager; NCCL collectives are graph-captured on
# a real multi-GPU node).  Timings are gloo/host-bound and not a bench result.
XG_BENCH_BACKEND=gloo python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port ${PORT:-29512} bench.py --gpus 2 --steps 3 --warmup 3
