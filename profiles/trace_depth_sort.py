"""Per-ticket phase timeline of the one-launch depth sort (tgs_debug_trace_depth_sort)
at c3 — used to find where each radix pass spends its time."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2501_14534_b200 import GaussianCloud, RenderSettings, _lib, render_forward, scenes  # noqa: E402

sc = scenes.config3(views=1)
st = RenderSettings(near=0.2, mask_threshold=0.01, sh_mask_threshold=0.1)
cloud = GaussianCloud.from_fields(sc.fields)
lib = _lib.load()
for _ in range(2):
    render_forward(cloud, sc.cameras[0], st)
buf = torch.zeros(8 * 4096, dtype=torch.int64, device="cuda")
lib.tgs_debug_trace_depth_sort(ctypes.c_void_p(buf.data_ptr()))
render_forward(cloud, sc.cameras[0], st)
torch.cuda.synchronize()
lib.tgs_debug_trace_depth_sort(ctypes.c_void_p(0))
tr = buf.view(-1, 8).cpu().numpy().astype(np.float64)
used = tr[:, 0] > 0
tr = tr[used]
t0 = tr[:, 0].min()
tr = np.where(tr > 0, (tr - t0) / 1e3, np.nan)  # us
n = len(cloud)
T0 = (n + 4095) // 4096
print(f"tickets used {used.sum()}, selection tiles {T0}")
sel = tr[:T0]
for k, name in enumerate(["start", "entered", "loaded+scanned", "looked back", "keys+hist", "done"]):
    print(f"selection {name:15s} min {np.nanmin(sel[:, k]):7.1f}  median {np.nanmedian(sel[:, k]):7.1f}  max {np.nanmax(sel[:, k]):7.1f} us")
for p in range(8):
    rows = tr[T0 + p * T0: T0 + (p + 1) * T0]
    live = rows[~np.isnan(rows[:, 5])]
    if not len(live):
        continue
    q = lambda k: (np.nanmin(live[:, k]), np.nanmedian(live[:, k]), np.nanmax(live[:, k]))
    print(f"pass {p}: tiles {len(live)}  start {q(0)[0]:.1f}/{q(0)[2]:.1f}  waited {q(1)[0]:.1f}/{q(1)[2]:.1f}  "
          f"loaded {q(2)[0]:.1f}/{q(2)[2]:.1f}  ranked {q(3)[0]:.1f}/{q(3)[2]:.1f}  "
          f"lookback {q(4)[0]:.1f}/{q(4)[1]:.1f}/{q(4)[2]:.1f}  done {q(5)[0]:.1f}/{q(5)[2]:.1f}")
