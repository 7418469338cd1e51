"""Time individual stages of the C2 step (CUDA events), no parity checks."""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_2512_16543_b200 import ops, scenario as S
dt = sys.argv[1] if len(sys.argv) > 1 else 'c128'
spec = S.C2.with_(dtype=dt)
dev = torch.device('cuda', 0)
H = torch.from_numpy(S.channels(spec)).to(dev)
B, T, K, N = H.shape
Hf = H.reshape(B * T, K, N)
G = ops.gram(Hf, spec.alpha)
Ainv, info = ops.herm_inverse(G)
noise = torch.full((B, K), spec.noise_var, dtype=torch.float64, device=dev)
def timeit(name, fn, n=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    print(f"{name:28s} {e0.elapsed_time(e1)/n:8.3f} ms")
timeit('gram', lambda: ops.gram(Hf, spec.alpha))
timeit('inverse', lambda: ops.herm_inverse(G))
timeit('precode (gram shortcut)', lambda: ops.precode_rate(Hf, Ainv, 1.0, noise, T, G_true=G, alpha=spec.alpha))
timeit('precode (H W)', lambda: ops.precode_rate(Hf, Ainv, 1.0, noise, T))
timeit('gram_delta formula', lambda: ops.gram_delta(Hf[:-1], Hf[1:], 1))
