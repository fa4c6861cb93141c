# The bench's N > 1 path (barriers, max over ranks, CeComm transport) on one GPU:
# two ranks time-slicing cuda:0 (TM_BENCH_SHARED_GPU=1); not a measurement.
set -u
TM_BENCH_SHARED_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config C3 --transport ce --steps 3 --warmup 3 --no-cpu 2>&1 | tail -2 | cut -c1-700
