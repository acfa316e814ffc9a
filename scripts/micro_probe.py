"""Single-thread cycle costs of the MMA warp's primitives (conv_q_micro_probe)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2202_06819_b200 as cq
lib = cq.load()
f = lib.conv_q_micro_probe
f.restype = ctypes.c_int
f.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
names = ["try_wait(done)", "test_wait(done)", "mma", "mma+commit", "commit", "stage: wait+4mma+commit",
         "stage: early try_wait", "empty loop", "elect+syncwarp", "asm memory clobber"]
for mode in range(10):
    row = []
    for n in (64, 128, 256):
        v = ctypes.c_double()
        rc = f(mode, 4000, n, ctypes.byref(v))
        row.append(f"N={n}: {v.value:7.1f}" if rc == 0 else f"N={n}: err")
    print(f"{names[mode]:28s} " + "  ".join(row), flush=True)
