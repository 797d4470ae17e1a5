"""Diagnostic: timeline of select_kernel's pair workers from %globaltimer
stamps (TLS_DEBUG_BUF): when each pair's last tile CTA starts, finishes its
tile, starts its worker (after the other tiles' flags), and how long the
top-k_b and the q-fragment / histogram setup take.  Not a bench line."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2604_07815_b200 as tls  # noqa: E402
from paper_2604_07815_b200 import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
bsz = int(sys.argv[2]) if len(sys.argv) > 2 else W.CONFIGS[name].batch
w = W.CONFIGS[name].with_(batch=bsz)
cfg, inputs, idx, queries = bench.build_state(w, 0, torch.device("cuda"), "outlier")
buf = torch.zeros(4 * 65536 * 8, dtype=torch.int64, device="cuda")
flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for it in range(3):
    if it == 2:
        os.environ["TLS_DEBUG_BUF"] = hex(buf.data_ptr())
    flush_buf.fill_(1)
    tls.decode(cfg, queries[it], inputs["k_cache"], inputs["v_cache"], inputs["seq_lens"], idx)
    torch.cuda.synchronize()
os.environ.pop("TLS_DEBUG_BUF")
pairs = w.batch * w.num_kv_heads
s = buf[: pairs * 16].view(pairs, 16).cpu().double() / 1e3  # us
t0 = s[:, 6].min()
def q(x):
    x = x.sort().values
    return f"min {float(x[0]):6.1f} med {float(x[len(x) // 2]):6.1f} max {float(x[-1]):6.1f}"
print(f"{w.name} pairs={pairs} (us, relative to the first worker-CTA start)")
print(f"  last-tile CTA start       {q(s[:, 6] - t0)}")
print(f"  own tile scored           {q(s[:, 8] - t0)}")
print(f"  worker start (flags seen) {q(s[:, 0] - t0)}")
print(f"  worker end                {q(s[:, 2] - t0)}")
print(f"  own tile: {q(s[:, 8] - s[:, 6])} | flag wait: {q(s[:, 0] - s[:, 8])}")
print(f"  top-k_b: {q(s[:, 1] - s[:, 0])} | q frags + hist zero: {q(s[:, 2] - s[:, 1])}")
print(f"    scores load {q(s[:, 3] - s[:, 0])} | fast_topk {q(s[:, 4] - s[:, 3])} | emit {q(s[:, 9] - s[:, 4])}"
      f" | sentinel restore {q(s[:, 1] - s[:, 9])}")
st = buf[65536 * 8: 65536 * 8 + 148 * 4].view(148, 4).cpu().double()
ok = st[:, 2] > 0
if ok.any():
    dur = (st[ok, 1] - st[ok, 0]) / 1e3
    print(f"  stream CTAs: {int(ok.sum())}, chunks each ~{float(st[ok, 2].median()):.0f}, duration {q(dur)} us, "
          f"start {q((st[ok, 0] - st[ok, 0].min()) / 1e3)}")
