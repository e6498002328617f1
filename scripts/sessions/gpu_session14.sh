#!/bin/bash
# P2 at 2^28 ring shapes around the policy; staged-batch tests (lazy items);
# the N>1 bench path on one GPU (gloo, same device)
TAG=${1:-r01v}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "batch or stage" > $OUT/pytest_batch.log 2>&1
for i in 1 2; do
  for cfg in "3 128 30" "3 128 32" "3 256 35" "3 256 34" "3 256 36" "3 192 30" "3 192 34" "4 128 28" "3 128 34"; do
    set -- $cfg
    TLK_STAGE=$1 TLK_STAGE_THREADS=$2 TLK_STAGE_READS=$3 timeout 300 python bench.py --no-e2e --no-cpu --no-configs --steps 20 > $OUT/bench_g$1x$2r$3_$i.json 2>> $OUT/bench_ab.err
  done
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 \
   bench.py --gpus 2 --dist-backend gloo --same-device --points 67108864 --steps 10 --warmup 3 --e2e-steps 1 \
   --no-cpu --no-configs > $OUT/bench_2rank_samedev.json 2> $OUT/bench_2rank_samedev.err
echo done > $OUT/DONE
