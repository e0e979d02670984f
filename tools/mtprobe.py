import ctypes as C, sys
sys.path.insert(0,'.')
import paper_2308_10169_b200 as pe
e = pe.Engine(0,'fp32')
f = pe.lib().sf_debug_mt_probe; f.restype=C.c_int; f.argtypes=[C.c_void_p, C.c_longlong, C.c_int, C.c_int, C.POINTER(C.c_double)]
for th in (320, 1024):
    for mode in (0,1,2,3,4,5):
        r = C.c_double()
        assert f(e._h, 2000, th, mode, C.byref(r)) == 0
        print("threads", th, "mode", mode, "cycles/block", round(r.value,1))
