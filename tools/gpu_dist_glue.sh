#!/bin/bash
# N > 1 glue of bench.py on ONE GPU: two ranks over gloo (CPU collectives); a
# functional check of the sharded path and its exactness check, never a measurement
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 \
  bench.py --gpus 2 --steps 2 --warmup 1 --rows 200000 --queries 1000 --dist-backend gloo --e2e-steps 1 > gpurun_out/dist_c2.json 2> gpurun_out/dist_c2.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518 \
  bench.py --config c5 --gpus 2 --steps 1 --warmup 1 --rows 4000000 --queries 512 --dist-backend gloo --e2e-steps 1 > gpurun_out/dist_c5.json 2> gpurun_out/dist_c5.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29519 \
  bench.py --config c5 --parallel query --gpus 2 --steps 1 --warmup 1 --rows 4000000 --queries 512 --dist-backend gloo --e2e-steps 1 > gpurun_out/dist_c5q.json 2> gpurun_out/dist_c5q.err
