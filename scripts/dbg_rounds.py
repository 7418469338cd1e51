"""Debug: screen-only rounds on C2 eta 0.9 -- how first_unverified advances."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2512_16543_b200 import ops, scenario as S
from paper_2512_16543_b200.omega import DeviceOmegaStreams, effective_i_max, normals_per_call_bound
dev = torch.device('cuda', 0)
B, T = 16, 200
spec = S.C2.with_(B=B, T=T)
eta = 0.9
trials = list(range(B))
H = torch.from_numpy(S.channels(spec, trials=trials)).to(dev)
K = spec.K
Hf = H.reshape(B * T, K, spec.N)
G = ops.gram(Hf, spec.alpha).reshape(B, T, K, K)
dA = torch.zeros(B, T, K, K, dtype=torch.complex128, device=dev)
dA[:, 1:] = G[:, 1:] - G[:, :-1]
dAf = dA.reshape(B * T, K, K)
st = DeviceOmegaStreams.for_method(spec.seed, eta, trials, dev)
L = T * normals_per_call_bound(K, spec.k_init, spec.p, spec.i_max, eta)
omega = st.window(L)
is_sketch = torch.ones(B, T, dtype=torch.uint8, device=dev); is_sketch[:, 0] = 0
i_eff = effective_i_max(K, spec.k_init, spec.p, spec.i_max, eta)
print('i_eff', i_eff, 'i_max', spec.i_max)
iters_pred = torch.full((B, T), i_eff, dtype=torch.int32, device=dev)
cursor = torch.zeros(B, T, dtype=torch.int64, device=dev)
cursor0 = torch.zeros(B, dtype=torch.int64, device=dev)
first = torch.zeros(B, dtype=torch.int32, device=dev)
active = torch.zeros(B, T, dtype=torch.uint8, device=dev)
pending = torch.zeros(1, dtype=torch.int32, device=dev)
votes = torch.empty(B, T, 16, dtype=torch.uint8, device=dev)
a = (is_sketch, iters_pred)
kw = (K, eta, spec.k_init, spec.p, spec.i_max)
ops.spec_verify(is_sketch, iters_pred, None, cursor, cursor0, first, active, pending, *kw, votes=votes)
D = ops.d_max_for(K, spec.k_init, spec.p, spec.i_max)
BT = B * T
res = dict(U=torch.empty(BT, D, K, dtype=torch.complex128, device=dev), V=torch.empty(BT, D, K, dtype=torch.complex128, device=dev),
           S=torch.zeros(BT, D, dtype=torch.float64, device=dev), k_est=torch.zeros(BT, dtype=torch.int32, device=dev),
           iters=torch.zeros(BT, dtype=torch.int32, device=dev), fallback=torch.zeros(BT, dtype=torch.int32, device=dev),
           consumed=torch.zeros(BT, dtype=torch.int64, device=dev))
row = torch.arange(B, dtype=torch.int32, device=dev).repeat_interleave(T)
for r in range(10):
    ops.arsvd(dAf, omega, cursor.reshape(BT), eta, spec.k_init, spec.p, spec.i_max, omega_row=row,
              mask=active.reshape(BT), out=res, want_factor=2, hermitian=True)
    it = res['iters'].reshape(B, T).cpu().numpy()
    pr = iters_pred.cpu().numpy()
    f0 = first.cpu().numpy()
    mism = [(int((it[b, f0[b]:] != pr[b, f0[b]:]).sum())) for b in range(B)]
    pending.zero_()
    ops.spec_verify(is_sketch, iters_pred, res['iters'], cursor, cursor0, first, active, pending, *kw, votes=votes)
    print('round', r, 'first', first.cpu().numpy().tolist(), 'mismatches in suffix', mism, 'active', int(active.sum()))
    if r == 0:
        print(' iters hist', np.unique(it[:, 1:], return_counts=True))
