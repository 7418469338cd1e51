import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2512_16543_b200 import leo as L, ops
cfg = L.ScenarioConfig().validate()
dev = torch.device("cuda", 0)
L.run_campaign(cfg.with_(mc_runs=2, pass_s=10.0), device=dev)
torch.cuda.synchronize()
ops.prof_enable(True, dev)
t = time.perf_counter()
res = L.run_campaign(cfg, device=dev)
torch.cuda.synchronize()
print("wall", time.perf_counter() - t)
for k, v in sorted(ops.prof_collect(dev).items(), key=lambda kv: -kv[1][0])[:15]:
    print(k, v)
