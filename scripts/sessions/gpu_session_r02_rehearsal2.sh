#!/bin/bash
# round-end rehearsal: exactly what the driver runs (pytest -m gpu, smoke, bench both arms)
TAG=${1:-r02rehearsal2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONPATH=$PWD
( time timeout 2400 python -m pytest tests -q -rs -m gpu ) > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
( time timeout 300 python -c "import __graft_entry__ as g; g.smoke()" ) > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
( time timeout 1200 python bench.py ) > $OUT/bench.json 2> $OUT/bench.err
( time timeout 900 python bench.py --impl reference ) > $OUT/bench_ref.json 2> $OUT/bench_ref.err
echo done > $OUT/DONE
