"""Calibration only (not product code): cuFFT batched complex128 throughput on
the lateral-pass shapes, to bound what the hand-written passes should reach."""
import torch

def t(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3

x = torch.randn(2 * 96 * 128, 256, dtype=torch.complex128, device="cuda")
us = t(lambda: torch.fft.fft(x, dim=-1))
print(f"contiguous 24576 x 256 fft: {us:.1f} us, {2 * x.numel() * 16 / us / 1e3:.0f} GB/s")
y = torch.randn(2 * 256, 256, 96, dtype=torch.complex128, device="cuda")  # [r*mx][my][plane]
us = t(lambda: torch.fft.fft(y, dim=1))
print(f"strided (my, plane-fastest) fft: {us:.1f} us, {2 * y.numel() * 16 / us / 1e3:.0f} GB/s")
z = torch.randn(2 * 96, 128, 128, dtype=torch.complex128, device="cuda")
us = t(lambda: torch.fft.fft2(z, s=(256, 256)))
print(f"padded 2-D fft2 192 x 128^2 -> 256^2: {us:.1f} us")
