#!/bin/bash
# block-local chunks (Variant.chunk) A/B on the BASELINE programs
OUT=${OUT:-gpurun_out/chunk}
mkdir -p $OUT
export PYTHONPATH=$PWD
CHUNKS=262144,2097152,33554432 ROUNDS=5 K=10 timeout 900 python scripts/tune_ab.py > $OUT/tune_ab_chunk.jsonl 2> $OUT/tune_ab_chunk.err
echo done > $OUT/DONE
