"""CTA-0 clock64 timeline of sf_mlp_fused (library built with -DSF_MLP_TRACE=1)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import mlp_bench  # noqa: E402,F401  (runs the timing once, leaves the trace of the last launch)
from paper_2511_22009_b200 import _lib  # noqa: E402

buf = np.zeros(16 * 64, dtype=np.int64)
assert ctypes.CDLL(_lib.LIB_PATH).sf_mlp_trace_read(buf.ctypes.data_as(ctypes.c_void_p)) == 0
tr = buf.reshape(16, 64)
t0 = tr[tr > 0].min()
names = ["fc1 start", "fc1 a1empty", "fc2 start", "fc2 hfull", "gelu a1full", "gelu hfull", "w take", "w full"]
names += ["P xfree ok", "P xempty ok", "E a2full", "E rfull", "E stats", "E done"]
print("i   " + " ".join(f"{n:>12s}" for n in names))
for i in range(48):
    print(f"{i:3d} " + " ".join(f"{(tr[r, i] - t0) if tr[r, i] else -1:12d}" for r in range(14)))
