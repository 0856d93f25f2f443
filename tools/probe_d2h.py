import mmap
import os
import sys
import time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_00688_b200 import _arrays as AR  # noqa: E402
x = torch.rand(4096, 256, 256, device="cuda")
n = x.numel() * 4
print(open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip(), torch.get_num_threads())
torch.cuda.synchronize()
for rep in range(3):
    t0 = time.perf_counter()
    out = torch.empty(tuple(x.shape), dtype=torch.float32)
    AR.download_into(out, x)
    t1 = time.perf_counter()
    mm = mmap.mmap(-1, n, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    mm.madvise(mmap.MADV_HUGEPAGE)
    out2 = torch.frombuffer(mm, dtype=torch.float32).view(x.shape)
    AR.download_into(out2, x)
    t2 = time.perf_counter()
    print(f"torch.empty+staged {t1-t0:.3f}s   mmap-hugepage+staged {t2-t1:.3f}s", flush=True)
    assert torch.equal(out, out2)
    del out, out2
