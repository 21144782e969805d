import sys, time, json
sys.path.insert(0, "/root/repo")
import torch
from paper_2510_00606_b200 import device as dev
a = torch.empty(5 << 30, dtype=torch.uint8, device="cuda")
b = torch.empty(5 << 30, dtype=torch.uint8, device="cuda")
for name, args in [("aligned4g", ([a.data_ptr()], [b.data_ptr()], [4 << 30], [False])),
                   ("mis1g", ([a.data_ptr() + (4 << 30) + 3], [b.data_ptr() + (4 << 30) + 8], [(1 << 30) - 16], [False])),
                   ("both", ([a.data_ptr(), a.data_ptr() + (4 << 30) + 3], [b.data_ptr(), b.data_ptr() + (4 << 30) + 8], [4 << 30, (1 << 30) - 16], [False, False]))]:
    p = dev.CopyProgram.from_pointers(*args)
    res = []
    for _ in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t = time.perf_counter()
        s.record(); p.launch(); e.record(); torch.cuda.synchronize()
        res.append((round(s.elapsed_time(e), 3), round((time.perf_counter() - t) * 1e3, 3)))
    print(name, res)
