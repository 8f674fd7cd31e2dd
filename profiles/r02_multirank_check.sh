# the N > 1 bench path (placement, routing, IPC peer pools, library-side directory, batched fetch) with
# two ranks sharing one GPU (not a scaling number; --pools random: materialised pools need ~89 GB per rank, one GPU each)
set -x
RC_BENCH_SHARE_GPU=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --pools random > gpurun_out/mr2.log 2>&1; echo mr=$?
tail -c 3000 gpurun_out/mr2.log
