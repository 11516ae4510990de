"""Print the CTA-0 clock64 timeline of one attention launch (library built with -DSF_ATTN_TRACE=1)."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_22009_b200 import _lib
rows, H, T = 128, 6, 1024
st = torch.cuda.current_stream().cuda_stream
q = (torch.randn(rows, H, T, 64, device="cuda") / 8).to(torch.bfloat16)
k = torch.randn(rows, H, T, 64, device="cuda").to(torch.bfloat16)
vt = torch.randn(rows, H, 64, T, device="cuda").to(torch.float16)
out = torch.empty(rows * T, H * 64, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    _lib.call("sf_attention", q.data_ptr(), k.data_ptr(), vt.data_ptr(), out.data_ptr(), rows, H, T, st)
torch.cuda.synchronize()
buf = np.zeros(16 * 64, dtype=np.int64)
lib = ctypes.CDLL(_lib.LIB_PATH)
assert lib.sf_attn_trace_read(buf.ctypes.data_as(ctypes.c_void_p)) == 0
tr = buf.reshape(16, 64)
t0 = tr[tr > 0].min()
names = ["A s_ready", "A p_done", "B s_ready", "B p_done", "A pv_issue", "A s_issue", "B pv_issue", "B s_issue",
         "A ld_done", "A max_done", "A p_comp", "A st_done", "B ld_done", "B max_done", "B p_comp", "B st_done"]
print("G   " + " ".join(f"{n:>11s}" for n in names))
for g in range(40):
    print(f"{g:3d} " + " ".join(f"{(tr[r, g] - t0) if tr[r, g] else -1:11d}" for r in range(16)))
