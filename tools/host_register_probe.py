import os, json, resource, sys
sys.path.insert(0, os.getcwd())
from multiprocessing import shared_memory
import torch
from paper_2510_00606_b200 import device as dev
torch.cuda.set_device(0)
print("memlock", resource.getrlimit(resource.RLIMIT_MEMLOCK), flush=True)
for gb in [2, 4, 6, 8, 12]:
    n = gb << 30
    shm = shared_memory.SharedMemory(name=f"regp{gb}", create=True, size=n)
    v = torch.frombuffer(shm.buf, dtype=torch.uint8)
    try:
        d = dev.host_register(v.data_ptr(), n); ok = True; dev.host_unregister(v.data_ptr())
    except Exception as e:
        ok = repr(e)[:80]
    # chunked
    okc = True
    try:
        regs = []
        for o in range(0, n, 1 << 30):
            regs.append(v.data_ptr() + o); p = dev.host_register(v.data_ptr() + o, min(1 << 30, n - o))
            if o == 0: first = p
        same = first == v.data_ptr()
        for a in regs: dev.host_unregister(a)
    except Exception as e:
        okc = repr(e)[:80]; same = None
    # prefault then register
    v.fill_(1)
    try:
        d = dev.host_register(v.data_ptr(), n); okf = True; dev.host_unregister(v.data_ptr())
    except Exception as e:
        okf = repr(e)[:80]
    print(json.dumps({"gb": gb, "whole": ok, "chunked_1g": okc, "dev_ptr_is_host_ptr": same, "prefaulted_whole": okf}), flush=True)
    del v; shm.close(); shm.unlink()
