"""C2 c128 Gram / fused precoder timing + error vs cuBLAS (torch) references.

    python scripts/dmma_probe.py            # DMMA kernels
    LRZ_SIMT_FP64=1 python scripts/dmma_probe.py   # SIMT DFMA kernels
"""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_16543_b200 import ops, scenario as S  # noqa: E402

dt = sys.argv[1] if len(sys.argv) > 1 else "c128"
spec = S.C2.with_(dtype=dt)
dev = torch.device("cuda", 0)
H = torch.from_numpy(S.channels(spec)).to(dev)
B, T, K, N = H.shape
Hf = H.reshape(B * T, K, N)
BT = B * T
mode = ("SIMT" if os.environ.get("LRZ_SIMT_FP64") == "1" else "DMMA") + " " + dt


def timeit(name, fn, n=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(f"{mode} {name:24s} {ms:8.3f} ms")
    return ms


G = ops.gram(Hf, spec.alpha)
Hd = Hf.to(torch.complex128)
Gref = Hd @ Hd.conj().transpose(-1, -2)
Gref = 0.5 * (Gref + Gref.conj().transpose(-1, -2))
Gref = Gref + spec.alpha * torch.eye(K, dtype=Gref.dtype, device=dev)
eg = ((G - Gref).abs().pow(2).sum((-1, -2)).sqrt() / Gref.abs().pow(2).sum((-1, -2)).sqrt()).max()
herm = (G - G.conj().transpose(-1, -2)).abs().max()
print(f"{mode} gram max rel err vs torch {eg.item():.2e}, hermitian defect {herm.item():.1e}")
Ainv, info = ops.herm_inverse(G)
noise = torch.full((B, K), spec.noise_var, dtype=torch.float64, device=dev)
W = torch.empty(BT, N, K, dtype=Hf.dtype, device=dev)
pr = ops.precode_rate(Hf, Ainv, 1.0, noise, T, W=W, G_true=G, alpha=spec.alpha)
Wref = Hd.conj().transpose(-1, -2) @ Ainv
ew = ((W - Wref).abs().pow(2).sum((-1, -2)).sqrt() / Wref.abs().pow(2).sum((-1, -2)).sqrt()).max()
s = 1.0 / Wref.abs().pow(2).sum((-1, -2)).sqrt()
C = (Hd @ Wref) * s[:, None, None]
P = C.abs() ** 2
sig = torch.diagonal(P, dim1=-2, dim2=-1)
q = sig / (P.sum(-1) - sig + spec.noise_var)
rates = torch.log2(1 + q)
er = ((pr["rates"] - rates).abs() / rates.abs()).max()
es = ((pr["scale"] - s).abs() / s).max()
print(f"{mode} precoder W rel err {ew.item():.2e}, rates {er.item():.2e}, scale {es.item():.2e}")
timeit("gram", lambda: ops.gram(Hf, spec.alpha))
timeit("precode_rate (W kept)", lambda: ops.precode_rate(Hf, Ainv, 1.0, noise, T, W=W,
                                                         G_true=G, alpha=spec.alpha))
timeit("precode_rate (W ws)", lambda: ops.precode_rate(Hf, Ainv, 1.0, noise, T, G_true=G,
                                                       alpha=spec.alpha, want_sinr=False))
timeit("inverse", lambda: ops.herm_inverse(G))
