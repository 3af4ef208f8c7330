"""Time sortPR on random_dfa(1e8, 4) with an arbitrary libdfm build (minimal ctypes,
old ABIs welcome): python tools/bisect_lib.py path/to/libdfm.so"""
import ctypes as C
import sys

lib = C.CDLL(sys.argv[1])
vp = C.c_void_p
ctx = vp()
assert lib.dfm_ctx_create(0, C.byref(ctx)) == 0
dd = vp()
lib.dfm_ddfa_random.argtypes = [vp, C.c_uint32, C.c_uint32, C.c_uint64, C.c_double, C.POINTER(vp)]
assert lib.dfm_ddfa_random(ctx, 100_000_000, 4, 1, 0.5, C.byref(dd)) == 0


class Lim(C.Structure):
    _fields_ = [("m", C.c_uint64), ("t", C.c_int64)]


buf = (C.c_char * 256)()
nb = C.c_uint32()
lim = Lim(16 << 30, 300000)
lib.dfm_run_algorithm_dev.argtypes = [vp, C.c_int32, vp, C.c_int32, C.POINTER(Lim), vp,
                                      C.POINTER(C.c_uint32), vp]
for _ in range(2):
    assert lib.dfm_run_algorithm_dev(ctx, 3, dd, 1, C.byref(lim), None, C.byref(nb), buf) == 0
print("blocks", nb.value)
