set -u
OUT=gpurun_out/r02d; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -rs -p no:cacheprovider -k "fused_program_matches or statement_by_statement or cross_domain or reference_harness or suite_statements" > $OUT/pytest_fixed.log 2>&1; echo "rc=$?" >> $OUT/pytest_fixed.log
timeout 600 python scripts/stream_probe.py > $OUT/stream_probe.jsonl 2> $OUT/stream_probe.err
cat > /tmp/tfill.py <<'PY'
import torch
a = torch.empty(1 << 30, dtype=torch.float64, device="cuda")
b = torch.empty(1 << 29, dtype=torch.float64, device="cuda")
for _ in range(2):
    a.fill_(1.5); b.copy_(a[: 1 << 29])
torch.cuda.synchronize()
PY
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__registers_per_thread,dram__bytes_write.sum,dram__bytes_read.sum --clock-control none --csv --log-file $OUT/ncu_torch_fill_copy.csv python /tmp/tfill.py > $OUT/ncu_torch.out 2>&1
timeout 600 ncu --set full --clock-control none -k regex:elementwise -c 1 -o $OUT/ncu_torch_fill python /tmp/tfill.py > $OUT/ncu_torch_full.out 2>&1
