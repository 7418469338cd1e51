"""Probe the arSVD front end on C2 Gram corrections: timing and hand-off counts."""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_2512_16543_b200 import ops, scenario as S
from paper_2512_16543_b200.omega import OmegaStreams, normals_per_call_max
spec = S.C2
B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
T = spec.T
dev = torch.device('cuda', 0)
H = torch.from_numpy(S.channels(spec.with_(B=B))).to(dev)
Hf = H.reshape(B * T, spec.K, spec.N)
dA = ops.gram_delta(Hf[:-1], Hf[1:], 1)
n = dA.shape[0]
L = normals_per_call_max(spec.K, spec.k_init, spec.p, spec.i_max)
om = torch.randn(n, L, dtype=torch.float64, device=dev)
cur = torch.zeros(n, dtype=torch.int64, device=dev)
for herm in (True, False):
    for rep in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        res = ops.arsvd(dA, om, cur, spec.eta, spec.k_init, spec.p, spec.i_max, want_factor=False, hermitian=herm)
        torch.cuda.synchronize(); t1 = time.perf_counter()
    ws = ops.workspace(dev, 0, 'arsvd')
    D = res['D']
    off = n * (2 * D * spec.K + D * D) * 16
    resume = ws[off:off + 4 * n].view(torch.int32).cpu().numpy()
    print('hermitian', herm, f'{(t1-t0)*1e3:.2f} ms', 'k hist', np.bincount(res['k_est'].cpu().numpy())[-3:],
          'fallback', res['fallback'].sum().item(), 'resumed' if herm else '', (resume >= 0).sum() if herm else '')
