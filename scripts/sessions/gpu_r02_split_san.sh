#!/bin/bash
# (1) fused P2 vs its two independent statements back to back (scripts/split_probe.py)
# (2) memcheck over the host-staged paths after the pageable detection moved to
#     cuPointerGetAttributes (no expected-error API reports)
OUT=${OUT:-gpurun_out/split}
mkdir -p $OUT
export PYTHONPATH=$PWD
timeout 900 python scripts/split_probe.py > $OUT/split_probe.jsonl 2> $OUT/split_probe.err
timeout 1500 compute-sanitizer --tool memcheck --target-processes all python -m pytest tests -q -x -m gpu \
  -k "pageable or concurrent_host or host_staged" > $OUT/sanitizer_host_memcheck.log 2>&1
echo "rc=$?" >> $OUT/sanitizer_host_memcheck.log
echo done > $OUT/DONE
