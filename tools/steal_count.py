import ctypes, sys, os
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_1203_5004_b200 import hood as H, workloads as W
L = H.library()
L.hood_internal_set_debug.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
L.hood_internal_steals.restype = ctypes.c_longlong
L.hood_internal_steals.argtypes = [ctypes.c_void_p]
ctx = H.Context.get(0)
for name, p, block in [("gauss26", W.gauss(1 << 26, seed=62), 0), ("arc25", W.arc(1 << 25), 0)]:
    t = torch.as_tensor(p).cuda()
    L.hood_internal_steals(ctx.handle)
    L.hood_internal_set_debug(ctx.handle, 4, None)
    rep = H.build_hood(t, block_len=block)
    s = L.hood_internal_steals(ctx.handle)
    L.hood_internal_set_debug(ctx.handle, 0, None)
    print(name, "steals", s, flush=True)
