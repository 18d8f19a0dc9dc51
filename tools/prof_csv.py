"""Per-kernel profile of one device-resident load_csv of the C2 table written
as CSV (tools/bench_next.py's CSV line): python tools/prof_csv.py"""
import ctypes as C
import sys
import time
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np
import torch
from paper_2403_05821_b200 import gen
from paper_2403_05821_b200._abi import PO_LOC_DEVICE, cuda_lib
from csv_util import to_csv

lib = cuda_lib()
text = to_csv(gen.generate(2))
d_text = torch.from_numpy(np.frombuffer(text, np.uint8).copy()).cuda()


def call():
    h = C.c_void_p(0)
    lib.check(lib.load_csv(d_text.data_ptr(), len(text), PO_LOC_DEVICE, C.byref(h), 0))
    lib.csv_free(h)


call()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    call()
torch.cuda.synchronize()
print("wall ms", (time.perf_counter() - t0) / 5 * 1e3, "bytes", len(text))
lib.profile_enable(1)
lib.profile_report()
call()
torch.cuda.synchronize()
prof = lib.profile_report()
for k, (c, ms) in sorted(prof.items(), key=lambda x: -x[1][1])[:10]:
    print(f"  {k:28s} {ms:8.3f} ms {c:4d}")
