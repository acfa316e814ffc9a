"""CTA 0 event timeline of one launch (instrumented build): per tile, when the
MMA warp got its accumulator buffer / first full stage / committed, and when
each epilogue warp got the accumulator / finished its store (clock64 cycles,
relative to the first producer event).
python scripts/timeline.py <layer|stem> <config> [N] [tiles to print]"""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("CONV_Q_LIB", os.path.join(ROOT, "paper_2202_06819_b200", "libconvq_instr.so"))
sys.path.insert(0, ROOT)
import torch
import paper_2202_06819_b200 as cq, workloads as wl
lib = cq.load()
lib.conv_q_plan_set_timeline.restype = ctypes.c_int
lib.conv_q_plan_set_timeline.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
name, cfg = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 256
show = int(sys.argv[4]) if len(sys.argv) > 4 else 12
g = wl.rng(9, 0)
if name == "stem":
    p = cq.StemPlan(N, 224, 224, 3, 64, 7, 7, 3, 8, relu=True)
    xd = torch.from_numpy(wl.random_bytes(g, p.x_dims)).cuda()
    wd = torch.from_numpy(wl.random_bytes(g, p.w_dims)).cuda()
    sd = torch.cat([torch.full((64,), 0.01), torch.zeros(64)]).cuda()
    y = torch.empty((N, 112, 112, 64), dtype=torch.uint8, device="cuda")
else:
    L = {l.name: l for l, _ in wl.resnet50_layers()}[name]
    x, w, ss = wl.layer_inputs(g, L, N, 8)
    p = cq.ConvPlan(N, L.H, L.W, L.C, L.K, L.R, L.S, L.stride, L.pad, 8, relu=True)
    xd, wd, sd = (torch.from_numpy(t).cuda() for t in (x, w, ss))
    y = torch.empty((N, L.P, L.Q, L.K), dtype=torch.uint8, device="cuda")
p.set_config(p.candidates().index(cfg))
for _ in range(3):
    p.run(xd, wd, sd, y)
tl = torch.zeros(64 * 256, dtype=torch.int64, device="cuda")
lib.conv_q_plan_set_timeline(p._h, ctypes.c_void_p(tl.data_ptr()))
p.run(xd, wd, sd, y)
torch.cuda.synchronize()
lib.conv_q_plan_set_timeline(p._h, None)
t = tl.view(64, 256).cpu()
base = int(t[0][t[0] > 0].min()) if (t[0] > 0).any() else int(t[t > 0].min())
def rel(v):
    return int(v) - base if int(v) > 0 else -1
ntiles = int((t[1] > 0).sum())
print(f"{name} {cfg}: CTA 0 ran {ntiles} tiles, producer stages {int((t[0] > 0).sum())}")
print("tile  acc_empty  full1  acc_commit | epilogue warps (got acc .. stored), cycles from first producer event")
epi = [w for w in range(20) if (t[4 + w] > 0).any()]
nb = len(set(int((t[4 + w] > 0).sum()) for w in epi))
for i in range(min(ntiles, show)):
    row = f"{i:4d} {rel(t[1][i]):9d} {rel(t[2][i]):7d} {rel(t[3][i]):9d} |"
    print(row)
print("producer stage events: " + " ".join(str(rel(t[0][i])) for i in range(min(int((t[0] > 0).sum()), 2 * show))))
# epilogue: per warp, its tiles' (acc, stored) pairs
for w in epi:
    k = int((t[4 + w] > 0).sum())
    pairs = [(rel(t[4 + w][j]), rel(t[24 + w][j])) for j in range(min(k, show))]
    print(f"  epi warp {w:2d}: " + " ".join(f"{a}..{b}" for a, b in pairs))
d = [rel(t[3][i + 1]) - rel(t[3][i]) for i in range(ntiles - 1)]
if d:
    d.sort()
    print(f"MMA commit-to-commit per tile: median {d[len(d)//2]} cycles, min {d[0]}, max {d[-1]}")
e = []
for w in epi:
    k = int((t[4 + w] > 0).sum())
    e += [rel(t[24 + w][j]) - rel(t[4 + w][j]) for j in range(k)]
if e:
    e.sort()
    print(f"epilogue warp busy per tile (acc -> stored): median {e[len(e)//2]} cycles, min {e[0]}, max {e[-1]}")
pr = [rel(t[0][i + 1]) - rel(t[0][i]) for i in range(int((t[0] > 0).sum()) - 1)]
if pr:
    pr.sort()
    print(f"producer stage-to-stage: median {pr[len(pr)//2]} cycles")
