"""Probe: does cuTensorMapEncodeTiled accept outer strides smaller than the inner extent?"""
import ctypes

import torch

torch.cuda.init()
x = torch.zeros(1 << 20, dtype=torch.bfloat16, device="cuda")
cu = ctypes.CDLL("libcuda.so.1")
f = cu.cuTensorMapEncodeTiled
f.restype = ctypes.c_int


def enc(inner, outer, stride_bytes, box_outer=128):
    tm = (ctypes.c_uint64 * 16)()
    dims = (ctypes.c_uint64 * 2)(inner, outer)
    strides = (ctypes.c_uint64 * 1)(stride_bytes)
    box = (ctypes.c_uint32 * 2)(64, box_outer)
    es = (ctypes.c_uint32 * 2)(1, 1)
    # dtype 10 = BFLOAT16, interleave 0, swizzle 3 = 128B, l2 promo 3 = 256B, oob 0
    return f(tm, 10, 2, ctypes.c_void_p(x.data_ptr()), dims, strides, box, es, 0, 3, 3, 0)


print("stride 128 (normal):", enc(64, 1000, 128))
print("stride 16 (overlap):", enc(64, 1000, 16))
print("stride 32 (overlap):", enc(64, 1000, 32))
