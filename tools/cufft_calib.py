"""Calibration only (not product): cuFFT (torch.fft) on the DST-shaped batches at n = 2048."""
import torch

dev = torch.device("cuda")
for L, batch in ((2047, 2048), (4094, 2048), (2048, 2048)):
    x = torch.randn(batch, L, dtype=torch.complex128, device=dev)
    xr = torch.randn(batch, L, dtype=torch.float64, device=dev)
    for name, f in (("c2c", lambda: torch.fft.fft(x, dim=1)), ("r2c", lambda: torch.fft.rfft(xr, dim=1))):
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            f()
        e1.record()
        torch.cuda.synchronize()
        print(f"cuFFT {name} L={L} batch={batch}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us")
