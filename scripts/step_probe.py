"""Where does a C2 bench step's time go?  Times the WB step with the Omega
window (a) generated on the main stream, (b) on a side stream, (c) reused
(no RNG), and the host time per step, with CUDA events over 10 steps."""

import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2512_16543_b200 import scenario as S  # noqa: E402
from paper_2512_16543_b200.omega import DeviceOmegaStreams  # noqa: E402
from paper_2512_16543_b200.trajectory import TrajectoryConfig, TrajectoryRunner  # noqa: E402

dev = torch.device("cuda", 0)
spec = S.C2
B, T, K, N = spec.B, spec.T, spec.K, spec.N
H = torch.from_numpy(S.channels(spec)).to(dev)
noise = torch.full((B, K), spec.noise_var, dtype=torch.float64, device=dev)
cfg = TrajectoryConfig(alpha=spec.alpha, eta=spec.eta, k_init=spec.k_init, p=spec.p,
                       i_max=spec.i_max)
st = DeviceOmegaStreams.for_method(spec.seed, spec.eta, range(B), dev)
side = torch.cuda.Stream(dev)
L = T * TrajectoryRunner(B, K, N, torch.complex128, cfg, dev).normals_per_step_max()
fixed = st.window(L).clone()


def step(mode):
    rn = TrajectoryRunner(B, K, N, torch.complex128, cfg, dev)
    st.raw.zero_()
    if mode == "main":
        om, ev = st.window(L), None
    elif mode == "side":
        om = st.window(L, stream=side)
        ev = st.ready
    else:
        om, ev = fixed, None
    return rn.run_chunk(H, noise, om, omega_ready=ev)


for mode in ("main", "side", "reuse", "main", "side", "reuse"):
    for _ in range(3):
        step(mode)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0 = time.perf_counter()
    e0.record()
    for _ in range(10):
        step(mode)
    e1.record()
    h1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"{mode:6s} gpu {e0.elapsed_time(e1) / 10:.3f} ms/step  host {1e3 * (h1 - h0) / 10:.3f} ms/step")
# host-side cost of issuing one step without the final sync wait
rn = TrajectoryRunner(B, K, N, torch.complex128, cfg, dev)
torch.cuda.synchronize()
