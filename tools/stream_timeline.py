"""Diagnostic: per-CTA timeline of stream_select_kernel (TLS_DEBUG_BUF stamps): start/end, SM, tiles, workers,
per-tile iteration start times.  Not a bench line.   python tools/stream_timeline.py c3"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2604_07815_b200 as tls  # noqa: E402
from paper_2604_07815_b200 import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
w = W.CONFIGS[name]
cfg, inputs, idx, queries = bench.build_state(w, 0, torch.device("cuda"), "outlier")
buf = torch.zeros(65536 * 32, dtype=torch.int64, device="cuda")  # the token / attention kernels stamp at 65536*16, *24
for it in range(4):
    if it == 3:
        buf.zero_()
        os.environ["TLS_DEBUG_BUF"] = hex(buf.data_ptr())
    tls.decode(cfg, queries[it % 8], inputs["k_cache"], inputs["v_cache"], inputs["seq_lens"], idx)
    torch.cuda.synchronize()
os.environ.pop("TLS_DEBUG_BUF", None)
print("nonzero words", int((buf != 0).sum()))
d = buf[: 296 * 256].view(296, 256).cpu().numpy()
d = d[d[:, 1] > 0]  # the streamers (the other CTA of each SM exits at once)
t0 = d[:, 0][d[:, 0] > 0].min()
st = (d[:, 0] - t0) / 1e3
en = (d[:, 1] - t0) / 1e3
print(f"{w.name}: streamers {int((d[:, 1] > 0).sum())}, start p0/50/100 {np.percentile(st, [0, 50, 100])}, "
      f"end p0/10/50/90/100 {np.percentile(en, [0, 10, 50, 90, 100])}")
sms = d[:, 2]
print("distinct SMs", len(set(sms.tolist())), "tiles per CTA", np.unique(d[:, 3], return_counts=True),
      "workers per CTA", np.unique(d[:, 4], return_counts=True))
ph = d[:, 8:248].reshape(-1, 60, 4).astype(np.int64)
st_ = (ph[:, :, 0] - t0) / 1e3
la = (ph[:, :, 1] - t0) / 1e3
ok = (ph[:, :, 0] > 0) & (ph[:, :, 1] > 0)
nxt = np.roll(st_, -1, axis=1)
okn = (ph[:, :, 0] > 0) & np.roll(ph[:, :, 0] > 0, -1, axis=1)
okn[:, -1] = False
pct = [10, 50, 90]
print("per slot (us) p10/50/90: start->rows landed", np.percentile((la - st_)[ok], pct),
      "slot period", np.percentile((nxt - st_)[okn], pct))
slow = np.argsort(-en)[:3]
for c in slow:
    print("slow CTA", c, "sm", d[c, 2], "end", en[c], "starts", np.round(st_[c, :10], 1))
