"""Batched Gram H H^H + alpha I for K in {16 .. 256}: DMMA vs SIMT kernels,
error against torch (cuBLAS) in complex128, timings.

    python scripts/gram_probe.py            # DMMA
    LRZ_SIMT_FP64=1 python scripts/gram_probe.py
"""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_16543_b200 import ops  # noqa: E402

dev = torch.device("cuda", 0)
mode = "SIMT" if os.environ.get("LRZ_SIMT_FP64") == "1" else "DMMA"
g = torch.Generator(device=dev)
g.manual_seed(1)
for K, N, B in ((16, 64, 4096), (40, 128, 2048), (64, 1024, 1024), (100, 512, 256),
                (128, 1024, 512), (256, 4096, 32)):
    for dt in (torch.complex64, torch.complex128):
        H = torch.randn(B, K, N, dtype=dt, device=dev, generator=g)
        G = ops.gram(H, 0.5)
        Hd = H.to(torch.complex128)
        R = Hd @ Hd.conj().transpose(-1, -2) + 0.5 * torch.eye(K, dtype=torch.complex128,
                                                                 device=dev)
        err = ((G - R).abs().pow(2).sum((-1, -2)).sqrt() / R.abs().pow(2).sum((-1, -2)).sqrt()).max()
        herm = (G - G.conj().transpose(-1, -2)).abs().max().item()
        ops.gram(H, 0.5)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(5):
            ops.gram(H, 0.5)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        tf = 4 * K * (K + 1) * N * B / (ms / 1e3) / 1e12
        print(f"{mode} K={K:3d} N={N:4d} B={B:5d} {str(dt)[-9:]}: rel err {err.item():.1e} "
              f"herm {herm:.0e}  {ms:7.3f} ms  {tf:5.1f} TF/s (algorithmic)")
