"""Intrinsic cost of the solve's 6-sum decision reduction on a c2 plan
(adp_debug_bench_reduce: the reduction run back to back in one launch)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402,F401
from paper_2502_09758_b200 import _native as nat  # noqa: E402

lib = nat.lib()
lib.adp_debug_bench_reduce.restype = ctypes.c_int
lib.adp_debug_bench_reduce.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.POINTER(ctypes.c_double), ctypes.c_void_p]
for shape, k in [((256, 256, 1), 9), ((512, 512, 3), 15)]:
    plan = nat.plan_for(nat.LAYOUT_DEPTHWISE2D, shape, (k, k))
    ms = ctypes.c_double()
    for reps in (10, 1000):
        nat.check(lib.adp_debug_bench_reduce(plan.handle, reps, ctypes.byref(ms), nat.stream_ptr()), "bench")
    nat.check(lib.adp_debug_bench_reduce(plan.handle, 1000, ctypes.byref(ms), nat.stream_ptr()), "bench")
    t1000 = ms.value
    nat.check(lib.adp_debug_bench_reduce(plan.handle, 10, ctypes.byref(ms), nat.stream_ptr()), "bench")
    print(shape, k, plan.geometry()["grid"], f"reduce: {(t1000 - ms.value) / 990 * 1e3:.2f} us each")
