"""Debug helper: row-copy mode vs the oracle on tiny stacks (prints mismatches)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import c_oracle as C  # noqa: E402
from paper_2211_00645_b200.deskew import deskew_device  # noqa: E402

for force in ("", "4", "2"):
    os.environ["SSB_FORCE_AC"] = force
    for (n, h, w, s, interp) in [(1, 3, 20, 0.0, "nearest"), (2, 2, 2, 1.0, "nearest"), (3, 4, 12, 0.7, "linear")]:
        st = (np.arange(n * h * w, dtype=np.uint16) + 1).reshape(n, h, w)
        raw = torch.from_numpy(st).cuda()
        res = deskew_device(raw, s, interp, reduce="max")
        torch.cuda.synchronize()
        want, _ = C.deskew(st, s, interp, reduce="max")
        got = res.volume.cpu().numpy()
        ok = (got == want).all()
        print("force", force or "-", (n, h, w, s, interp), "ok" if ok else "MISMATCH")
        if not ok and n == 1:
            print("got\n", got, "\nwant\n", want)
