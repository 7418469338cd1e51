"""Batched Hermitian inverse timing and redo-flag count per K."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2512_16543_b200 import ops
dev = torch.device("cuda", 0)
for K, B in ((32, 12800), (64, 12800), (128, 8192), (256, 640)):
    g = torch.Generator(device=dev).manual_seed(0)
    X = torch.randn(B, K, 2 * K, dtype=torch.complex128, device=dev, generator=g)
    A = X @ X.mH + 0.5 * torch.eye(K, dtype=torch.complex128, device=dev)
    out, info = ops.herm_inverse(A)
    torch.cuda.synchronize()
    ws = ops._WS.get((0, torch.cuda.current_stream(dev).cuda_stream, "inv"))
    nredo = int(ws[:B].sum().item()) if ws is not None else -1
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        ops.herm_inverse(A, out=out, info=info)
    e1.record()
    torch.cuda.synchronize()
    err = (A[:4] @ out[:4] - torch.eye(K, dtype=torch.complex128, device=dev)).abs().max().item()
    print(f"K={K} B={B}: {e0.elapsed_time(e1) / 3:.3f} ms, redo {nredo}, max|A A^-1 - I| {err:.1e}")
