import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2202_06819_b200 as cq
lib = cq.load()
for f in (lib.conv_q_mma_pipe_probe, lib.conv_q_mma_pipe_probe2):
    f.restype = ctypes.c_int
    f.argtypes = [ctypes.c_int] * 4 + [ctypes.POINTER(ctypes.c_double)]
for name, f in (("cta1 M=128", lib.conv_q_mma_pipe_probe), ("pair M=256", lib.conv_q_mma_pipe_probe2)):
    for n in (256, 128, 64):
        for G in (2, 4, 8, 16):
            row = []
            for S in (1, 2, 3, 4, 8):
                v = ctypes.c_double()
                groups = max(64, 100000 // G)
                rc = f(groups, G, S, n, ctypes.byref(v))
                row.append(f"S{S}:{v.value/1e12:6.0f}" if rc == 0 else f"S{S}:err")
            print(f"{name} N={n:3d} G={G:2d}  " + "  ".join(row), flush=True)
