import torch, time, sys
sys.path.insert(0, ".")
from paper_2512_16543_b200.omega import DeviceOmegaStreams
d = torch.device("cuda", 0)
st = DeviceOmegaStreams.for_method(0, 0.999, list(range(64)), d)
for i in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    st.raw.zero_(); w = st.window(640000)
    torch.cuda.synchronize(); print("window ms", (time.perf_counter() - t) * 1e3)
