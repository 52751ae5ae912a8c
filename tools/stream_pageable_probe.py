"""StackStreamer.run throughput from pinned vs pageable host stacks (config-2 size, no volume D2H)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2211_00645_b200.stream import StackStreamer, pinned_stack  # noqa: E402

n, h, w, s = 512, 2048, 2048, 0.8660254037844386
pin = pinned_stack(n, h, w)
pin[:] = np.random.default_rng(0).integers(0, 4096, size=(n, h, w), dtype=np.uint16)
pageable = np.array(pin)
streamer = StackStreamer(h, w)
for label, src in (("pinned", pin), ("pageable", pageable)):
    res = streamer.run(src, s, "linear", write_volume=False)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        res = streamer.run(src, s, "linear", write_volume=False)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) / 3 * 1e3
    print(json.dumps({"host": label, "ms_per_stack": ms, "GBps": 2 * n * h * w / ms / 1e6,
                      "torch_threads": torch.get_num_threads()}), flush=True)
