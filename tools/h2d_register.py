import time, numpy as np, torch, ctypes
cu = ctypes.CDLL("libcudart.so.12") if False else None
import torch.cuda
rt = torch.cuda.cudart()
a = np.ones(1 << 28, dtype=np.float64)  # 2 GiB
d = torch.empty(1 << 28, dtype=torch.float64, device="cuda")
for it in range(3):
    t0 = time.perf_counter()
    r = rt.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
    t1 = time.perf_counter()
    d.copy_(torch.from_numpy(a), non_blocking=False)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    rt.cudaHostUnregister(a.ctypes.data)
    t3 = time.perf_counter()
    print("register", r, f"{(t1-t0)*1e3:.1f} ms ({a.nbytes/(t1-t0)/1e9:.1f} GB/s) copy {(t2-t1)*1e3:.1f} ms unregister {(t3-t2)*1e3:.1f} ms", flush=True)
b = np.empty_like(a)
for th in (1,):
    t0 = time.perf_counter(); np.copyto(b, a); t1 = time.perf_counter()
    print(f"numpy memcpy 1 thread {a.nbytes/(t1-t0)/1e9:.1f} GB/s")
