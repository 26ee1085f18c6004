set -x
OUT=gpurun_out/g50
mkdir -p $OUT
python - > $OUT/probe.txt 2>&1 <<'PY'
import torch, time
h = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True); d = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
for i in range(12):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        a.record(); d.copy_(h, non_blocking=True); b.record()
    b.synchronize(); print(round((1 << 30) / (a.elapsed_time(b) * 1e-3) / 1e9, 2))
PY
nvidia-smi -q -d PCIE > $OUT/pcie.txt 2>&1
for r in 1 2; do
  timeout 600 python bench.py > $OUT/bench_default_$r.json 2> $OUT/bench_default_$r.log
done
