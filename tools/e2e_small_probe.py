import math, time, sys, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from paper_2211_00645_b200.stream import StackStreamer, pinned_stack
n,h,w = 128,256,512
s = math.cos(math.radians(30))
host = pinned_stack(n,h,w); host[:] = np.random.default_rng(0).integers(0,4096,(n,h,w)).astype(np.uint16)
st = StackStreamer(h, w)
for _ in range(3): r = st.run(host, s, "linear"); del r
torch.cuda.synchronize()
for k in range(5):
    t0=time.perf_counter(); e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record(); r = st.run(host, s, "linear"); e1.record(); torch.cuda.synchronize(); t1=time.perf_counter()
    print(f"run: wall {1e3*(t1-t0):.3f} ms, events {e0.elapsed_time(e1):.3f} ms, host part {st.timings.total_ms:.3f} ms"); del r
import torch.profiler as tp
with tp.profile(activities=[tp.ProfilerActivity.CPU, tp.ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        r = st.run(host, s, "linear"); del r
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=12))
