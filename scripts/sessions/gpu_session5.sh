#!/bin/bash
# full parity suite, smoke, bench both arms, and compute-sanitizer on the kernels
TAG=${1:-r01h}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONPATH=$PWD
timeout 1500 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
# memcheck (flat, batch, host-staged paths) and racecheck (batch entry: shared-memory staging)
timeout 900 compute-sanitizer --tool memcheck --target-processes all python -m pytest tests/test_gpu_parity.py -q -x \
   -k "fused_program_matches_reference_bitwise and (c4_p2 or c4_p3 or special or aliased or c1_dtg_odd) or multi_domain_batch or ragged or host_fields_staged and c4_p3" \
   > $OUT/sanitizer_memcheck.log 2>&1; echo "memcheck rc=$?" >> $OUT/sanitizer_memcheck.log
timeout 900 compute-sanitizer --tool racecheck --target-processes all python -m pytest tests/test_gpu_parity.py -q -x \
   -k "multi_domain_batch or ragged" > $OUT/sanitizer_racecheck.log 2>&1; echo "racecheck rc=$?" >> $OUT/sanitizer_racecheck.log
echo done > $OUT/DONE
