"""One WB chunk of a BASELINE config (device channels + device Omega), for ncu.

    python scripts/prof_cfg.py C5 c128 [chunk] [B] [eta]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2512_16543_b200 import scenario as S  # noqa: E402
from paper_2512_16543_b200.omega import DeviceOmegaStreams  # noqa: E402
from paper_2512_16543_b200.trajectory import TrajectoryConfig, TrajectoryRunner  # noqa: E402

name, dt = sys.argv[1], sys.argv[2]
chunk = int(sys.argv[3]) if len(sys.argv) > 3 else 25
spec = S.CONFIGS[name].with_(dtype=dt)
if len(sys.argv) > 4:
    spec = spec.with_(B=int(sys.argv[4]))
eta = float(sys.argv[5]) if len(sys.argv) > 5 else spec.eta
dev = torch.device("cuda", 0)
trials = list(range(spec.B))
chans = S.DeviceChannels(spec, trials, dev)
tdt = torch.complex64 if dt == "c64" else torch.complex128
noise = torch.full((spec.B, spec.K), spec.noise_var, dtype=torch.float64, device=dev)
cfg = TrajectoryConfig(alpha=spec.alpha, eta=eta, k_init=spec.k_init, p=spec.p,
                       i_max=spec.i_max)
rn = TrajectoryRunner(spec.B, spec.K, spec.N, tdt, cfg, dev)
st = DeviceOmegaStreams.for_method(spec.seed, eta, trials, dev)
for c in range(min(2, max(1, spec.T // chunk))):
    H = chans.generate(c * chunk, (c + 1) * chunk)
    om = st.window(chunk * rn.normals_per_step_max())
    r = rn.run_chunk(H, noise, om)
    st.advance(r.consumed)
torch.cuda.synchronize()
print("ok", name, dt, r.method.float().mean().item())
