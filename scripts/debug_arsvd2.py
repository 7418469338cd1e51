import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2512_16543_b200 import ops
from paper_2512_16543_b200.omega import normals_per_call_max
np.set_printoptions(precision=2, linewidth=200)
g = np.load('tests/golden/arsvd_cases.npz')
ci, eta, p = 6, 0.999, 5
dA = g[f"c{ci}_dA"]; K = dA.shape[0]
srng = np.random.default_rng([ci, int(eta * 1000), p, 4])
z = srng.standard_normal(normals_per_call_max(K, 2, p, 4))
dev = torch.device('cuda', 0)
t = torch.from_numpy(dA).to(dev)[None].contiguous()
om = torch.from_numpy(z).to(dev)[None].contiguous()
cur = torch.zeros(1, dtype=torch.int64, device=dev)
res = ops.arsvd(t, om, cur, eta, 2, p, 1)
torch.cuda.synchronize()
D = res['D']; d = 7
ws = ops.workspace(dev, 0, 'arsvd')
w = ws[:(2 * D * K + D * D) * 16].view(torch.complex128).cpu().numpy()
Q = w[:D * K].reshape(D, K).T[:, :d]
print(np.abs(Q.conj().T @ Q))
print(np.linalg.norm(Q, axis=0))
SQH = np.sqrt(0.5)
Om = SQH * (z[:K * d].reshape(K, d) + 1j * z[K * d:2 * K * d].reshape(K, d))
Y = dA @ Om
print('Y col norms', np.linalg.norm(Y, axis=0))
print('rank-1 residuals', [np.linalg.norm(Y[:, j] - Q[:, 0] * (Q[:, 0].conj() @ Y[:, j])) for j in range(d)])
