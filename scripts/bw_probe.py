"""Write / copy bandwidth ceilings for the label write (development probe)."""
import torch
H = W = 21600
n = H * W
lab = torch.empty(n, dtype=torch.int32, device="cuda")
img = torch.empty(n, dtype=torch.uint8, device="cuda")
def t(f, reps=20):
    for _ in range(3): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
ms = t(lambda: lab.fill_(7))
print(f"fill int32 {n*4/1e9:.2f} GB: {ms*1000:.1f} us = {n*4/ms/1e6:.0f} GB/s")
ms = t(lambda: lab.copy_(img))
print(f"u8->int32 convert copy ({n*5/1e9:.2f} GB): {ms*1000:.1f} us = {n*5/ms/1e6:.0f} GB/s")
ms = t(lambda: img.fill_(1))
print(f"fill u8 {n/1e9:.2f} GB: {ms*1000:.1f} us = {n/ms/1e6:.0f} GB/s")
