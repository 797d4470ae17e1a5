"""Diagnostic: per-item timeline of the persistent step kernel (pstep.cu) from
its %globaltimer stamps (TLS_DEBUG_BUF): for every ticket (start, end, SM,
role, sub).  Prints per-role item durations and, per role, when the items ran
(start/end percentiles) plus the busy time per SM.  Not a bench line.
    python tools/pstep_timeline.py c3 [_ [batch]]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2604_07815_b200 as tls  # noqa: E402
from paper_2604_07815_b200 import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
os.environ.setdefault("TLS_PSTEP", "1")
w = W.CONFIGS[name]
if len(sys.argv) > 3:
    w = w.with_(batch=int(sys.argv[3]))
cfg, inputs, idx, queries = bench.build_state(w, 0, torch.device("cuda"), "outlier")
buf = torch.zeros((1 << 20) + 1 + 8192, dtype=torch.int64, device="cuda")
flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
times = []
ALWAYS = os.environ.get("DBG_ALWAYS") == "1"
for it in range(8):
    if it == 7 or ALWAYS:
        buf.zero_()
        os.environ["TLS_DEBUG_BUF"] = hex(buf.data_ptr())
    flush_buf.fill_(1)
    ev[0].record()
    tls.decode(cfg, queries[it % 8], inputs["k_cache"], inputs["v_cache"], inputs["seq_lens"], idx)
    ev[1].record()
    torch.cuda.synchronize()
    times.append(ev[0].elapsed_time(ev[1]) * 1e3)
os.environ.pop("TLS_DEBUG_BUF", None)
hung = int(buf[1 << 20].item())
if hung:
    info = buf[(1 << 20) + 1:(1 << 20) + 1 + 2 * min(hung, 4096)].view(-1, 2).cpu().numpy()
    print(f"HUNG WAITS: {hung}")
    for tag, val in info[:40]:
        print(f"  pair {tag >> 32} kind {(tag >> 16) & 0xff} sub {tag & 0xffff}: observed {val >> 32} want {val & 0xffffffff}")
raw = buf[: 3 * ((1 << 20) // 3)].view(-1, 3).cpu().numpy()
raw = raw[raw[:, 1] > 0]
t0 = raw[:, 0].min()
st = (raw[:, 0] - t0) / 1e3
en = (raw[:, 1] - t0) / 1e3
role = (raw[:, 2] >> 24) & 0xff
sm = raw[:, 2] >> 32
print(f"{w.name}: step us (no stamps) {np.median(times[:7]):.1f}, with stamps {times[7]:.1f}; tickets {len(raw)}")
names = ["TILE", "TOKEN", "SEL", "ATT"]
pct = (0, 10, 50, 90, 100)
for r, nm in enumerate(names):
    sel = role == r
    if not sel.any():
        continue
    dur = en[sel] - st[sel]
    print(f"  {nm:6s} n={sel.sum():5d} dur us " + " ".join(f"{np.percentile(dur, p):6.1f}" for p in pct) +
          " | start " + " ".join(f"{np.percentile(st[sel], p):6.1f}" for p in pct) +
          " | end " + " ".join(f"{np.percentile(en[sel], p):6.1f}" for p in pct) +
          f" | CTA-us {dur.sum():8.0f}")
busy = np.zeros(int(sm.max()) + 1)
for s_, a, b in zip(sm, st, en):
    busy[s_] += b - a
print(f"  end {en.max():.1f} us; busy CTA-us per SM: median {np.median(busy):.0f}, max {busy.max():.0f}")
# per-tile stamps of run_tiles (dbg[2^19 + 3 t]: issue, first rows landed, scored)
ts = buf[(1 << 19):(1 << 19) + 3 * 20000].view(-1, 3).cpu().numpy().astype(np.int64)
ts = ts[(ts[:, 0] > 0) & (ts[:, 2] > 0)]
if len(ts):
    lat = (ts[:, 1] - ts[:, 0]) / 1e3
    cmp_ = (ts[:, 2] - ts[:, 1]) / 1e3
    print(f"  tiles {len(ts)}: issue->landed us " + " ".join(f"{np.percentile(lat, p):6.2f}" for p in pct) +
          " | landed->scored " + " ".join(f"{np.percentile(cmp_, p):6.2f}" for p in pct))
    iss = np.sort((ts[:, 0] - t0) / 1e3)
    print("  tile issue times us p0..p100: " + " ".join(f"{np.percentile(iss, p):6.1f}" for p in pct))
