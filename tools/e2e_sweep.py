"""Times wf_session_run_host (pinned host buffers) for several chunk sizes."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2107_11983_b200 import engine as E  # noqa: E402
from paper_2107_11983_b200.host import ExecOptions, QuerySpec  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else "c2"]
dg = E.DeviceGraph.rmat(cfg["scale"], 16, seed=1, weighted=cfg["weighted"], label_count=cfg["labels"])
V = dg.info()["V"]
spec, lo, hi = bench.query_plan(cfg, V, 0, 1)
n = hi - lo
stride = bench.row_capacity(cfg)
sess = E.Session(dg, bench.program_of(cfg), ExecOptions(seed=1, path_stride=stride))
if "--tune" in sys.argv:
    d_src = torch.from_numpy(spec.sources.view(np.int32)).cuda()
    print("tuned blocks/SM, ms:", sess.tune(spec, lo, hi, sources_dev_ptr=d_src.data_ptr()))
h_src = torch.from_numpy(spec.sources.view(np.int32)).pin_memory()
hspec = QuerySpec.from_list(h_src.numpy().view(np.uint32))
cap = n * stride
h_off = torch.empty(n + 1, dtype=torch.int64).pin_memory()
h_vert = torch.empty(cap, dtype=torch.int32).pin_memory()
h_stat = torch.empty(n, dtype=torch.uint8).pin_memory()
chunks = [0, 1 << 17, 1 << 18, 3 << 17, 1 << 19, 3 << 18, 1 << 20, 1 << 21]
for a in sys.argv:
    if a.startswith("--chunks="):
        chunks = [int(x) for x in a.split("=", 1)[1].split(",")]
for chunk in chunks:
    if chunk > n:
        continue
    ts = []
    records = "--records" in sys.argv
    h_rec = torch.empty(n, dtype=torch.int32).pin_memory() if records else None
    for _ in range(5):
        t = time.perf_counter()
        if records:
            m = sess.run_host_records(hspec, h_rec.data_ptr(), h_vert.data_ptr(), cap, chunk=chunk)
        else:
            m = sess.run_host(hspec, h_off.data_ptr(), h_vert.data_ptr(), cap, h_stat.data_ptr(), chunk=chunk)
        ts.append(time.perf_counter() - t)
    best = min(ts[1:])
    nv = int((h_rec.numpy().view(np.uint32) & 0x7FFFFFFF).astype(np.int64).sum()) if records else int(h_off[n].item())
    h_off[n] = nv
    print(f"chunk {chunk}: {best*1e3:.3f} ms  {m.total_steps/best/1e9:.2f} G steps/s  "
          f"bytes {nv*4 + (n * 4 if records else (n+1)*8 + n)}", flush=True)
# raw PCIe D2H of the same bytes for reference
nbytes = int(h_off[n].item()) * 4
d = torch.empty(nbytes // 4, dtype=torch.int32, device="cuda")
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    h_vert[: nbytes // 4].copy_(d, non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t) / 5
print(f"plain D2H of {nbytes/1e6:.1f} MB: {dt*1e3:.3f} ms = {nbytes/dt/1e9:.1f} GB/s")
