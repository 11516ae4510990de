import os, sys, torch, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2511_22009_b200 as sf
S, D = 256, 16384
seeds = torch.arange(1000, 1000 + S, dtype=torch.int64, device="cuda")
out = torch.empty(S, D, dtype=torch.float64, device="cuda")
for g in range(3):
    sf.numpy_noise_device(seeds, g, D, out=out)
torch.cuda.synchronize()
print("ok")
