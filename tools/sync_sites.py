"""Stream syncs of one device-resident ggr() call by call site
(PO_DEBUG_SYNCS=1 prints them to stderr): python tools/sync_sites.py cfg rows."""
import os
import subprocess
import sys
from collections import Counter

if os.environ.get("PO_DEBUG_SYNCS") != "1":
    env = dict(os.environ, PO_DEBUG_SYNCS="1")
    r = subprocess.run([sys.executable, __file__] + sys.argv[1:], env=env, capture_output=True, text=True)
    lines = [l for l in r.stderr.splitlines() if l.startswith("[po sync]")]
    mark = [i for i, l in enumerate(r.stderr.splitlines()) if l.startswith("=== measured")]
    all_lines = r.stderr.splitlines()
    start = mark[0] if mark else 0
    sites = [l.split()[-1] for l in all_lines[start:] if l.startswith("[po sync]")]
    print(f"{len(sites)} syncs in the measured call")
    for k, v in Counter(s.split("/")[-1] for s in sites).most_common():
        print(f"  {v:3d}  {k}")
    sys.exit(0)
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2403_05821_b200 as po
from paper_2403_05821_b200 import gen
from paper_2403_05821_b200._abi import PO_LOC_DEVICE

cfg_id, rows = int(sys.argv[1]), int(sys.argv[2])
t = gen.generate(cfg_id, n_rows=rows)
n, m = t.row_count(), t.field_count()
fd = [[t.require_field(x) for x in g] for g in gen.fds(cfg_id)]
dv = t.view(PO_LOC_DEVICE, arena=torch.from_numpy(t.arena).cuda(),
            offsets=torch.from_numpy(t.offsets.view(np.int64)).cuda())
r_ = torch.empty(n, dtype=torch.int64, device="cuda")
o_ = torch.empty(n * m, dtype=torch.int32, device="cuda")
po.ggr_into(dv, fd, po.GgrConfig(), 0, 0, PO_LOC_DEVICE, r_, o_, 0)
torch.cuda.synchronize()
print("=== measured", file=sys.stderr, flush=True)
po.ggr_into(dv, fd, po.GgrConfig(), 0, 0, PO_LOC_DEVICE, r_, o_, 0)
torch.cuda.synchronize()
