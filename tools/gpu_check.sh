set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
python - <<'PY' > gpurun_out/l2probe.txt 2>&1
import torch, time
x = torch.empty(64*1024*1024//2, dtype=torch.bfloat16, device='cuda'); y = torch.empty_like(x)
for sz_mb in [16, 32, 48, 64, 96, 2048]:
    a = torch.empty(sz_mb*1024*1024//4, dtype=torch.float32, device='cuda'); b = torch.empty_like(a)
    for _ in range(3): b.copy_(a)
    torch.cuda.synchronize(); e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record(); 
    for _ in range(50): b.copy_(a)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)/50
    print(f"copy {sz_mb} MB: {2*a.numel()*4/ms/1e6:.0f} GB/s (read+write)")
    # read-only: sum
    e0.record()
    for _ in range(50): a.sum()
    e1.record(); torch.cuda.synchronize(); ms = e0.elapsed_time(e1)/50
    print(f"sum  {sz_mb} MB: {a.numel()*4/ms/1e6:.0f} GB/s (read)")
PY
cat gpurun_out/l2probe.txt
timeout 600 python -m pytest tests/test_tc_probe.py -q 2>&1 | tail -15
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "not full_size" 2>&1 | tail -30
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -3
timeout 600 python bench.py --steps 2 --warmup 3 --n 32768 --no-cpu 2>&1 | tail -3
