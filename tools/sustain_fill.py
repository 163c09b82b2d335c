import torch, time, json, subprocess
x = torch.empty(12 * 2**30 // 8, dtype=torch.float64, device="cuda")
ts = []
for i in range(60):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); x.fill_(1.0 + i); b.record(); b.synchronize()
    ts.append(a.elapsed_time(b))
gb = x.numel() * 8 / 1e9
print("fill GB/s per iter:", [round(gb / t * 1e3) for t in ts[::5]])
print(subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,power.draw,clocks_throttle_reasons.active", "--format=csv"], capture_output=True, text=True).stdout)
