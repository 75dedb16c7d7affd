#!/bin/bash
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/peaks_clocks.csv &
SMI=$!
./tools/fp64_peaks > gpurun_out/fp64_peaks.json 2>&1
python - <<'PY' >> gpurun_out/fp64_peaks_torch.txt 2>&1
import torch, time
a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
b = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
for _ in range(2): a @ b
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
best = 1e9
for _ in range(5):
    e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
print("dgemm_8192_tflops", 2 * 8192**3 / (best * 1e-3) / 1e12)
PY
kill $SMI
nvidia-smi -q | grep -i -A3 "Clocks" | head -20 >> gpurun_out/fp64_peaks_torch.txt
