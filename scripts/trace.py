"""Per-CTA wait attribution for a layer/config: python scripts/trace.py l3.b1.c2 [config...]"""
import ctypes, os, sys
# measurement build (CONVQ_INSTRUMENT=1 python paper_2202_06819_b200/_build.py)
os.environ.setdefault("CONV_Q_LIB", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2202_06819_b200", "libconvq_instr.so"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2202_06819_b200 as cq, workloads as wl
lib = cq.load()
lib.conv_q_plan_set_trace.restype = ctypes.c_int
lib.conv_q_plan_set_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
name = sys.argv[1]
net = os.environ.get("TRACE_NET", "resnet50")
N, bits = int(os.environ.get("TRACE_N", 256)), int(os.environ.get("TRACE_BITS", 8))
g = wl.rng(9, 0)
if name == "stem":   # ResNet conv1 through the s2d StemPlan
    p = cq.StemPlan(N, 224, 224, 3, 64, 7, 7, 3, bits, relu=True)
    xd = torch.from_numpy(wl.random_bytes(g, p.x_dims)).cuda()
    wd = torch.from_numpy(wl.random_bytes(g, p.w_dims)).cuda()
    sd = torch.cat([torch.full((64,), 0.01), torch.zeros(64)]).cuda()
    y = torch.empty((N, 112, 112, 64 * bits // 8), dtype=torch.uint8, device="cuda")
else:
    L = {l.name: l for l, _ in getattr(wl, net + "_layers")()}[name]
    x, w, ss = wl.layer_inputs(g, L, N, bits)
    p = cq.ConvPlan(N, L.H, L.W, L.C, L.K, L.R, L.S, L.stride, L.pad, bits, relu=True)
    xd, wd, sd = (torch.from_numpy(t).cuda() for t in (x, w, ss))
    y = torch.empty((N, L.P, L.Q, L.K * bits // 8), dtype=torch.uint8, device="cuda")
cfgs = sys.argv[2:] or p.candidates()
names = ["prod_wait_empty", "mma_wait_full", "mma_wait_acc", "epi_wait_acc", "mma_issue", "total", "tiles"]
enames = ["epi_slab", "epi_body", "epi_store"]
for cname in cfgs:
    p.set_config(p.candidates().index(cname))
    for _ in range(3): p.run(xd, wd, sd, y)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(10): p.run(xd, wd, sd, y)
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 10 * 1000
    tr = torch.zeros(148 * 15, dtype=torch.int64, device="cuda")
    h0, h1 = torch.cuda.Event(True), torch.cuda.Event(True)
    lib.conv_q_plan_set_trace(p._h, ctypes.c_void_p(tr.data_ptr()))
    torch.cuda.synchronize()
    h0.record()
    p.run(xd, wd, sd, y)
    h1.record()
    torch.cuda.synchronize()
    lib.conv_q_plan_set_trace(p._h, None)
    t = tr.view(148, 15).double().cpu()
    act = t[:, 5] > 0
    m = t[act].mean(0)
    s = "  ".join(f"{n}={m[i]/1965:6.1f}" for i, n in enumerate(names[:6]))
    s += "  " + "  ".join(f"{n}={m[12 + i]/1965:6.1f}" for i, n in enumerate(enames))
    t0 = t[act, 7]; t1 = t[act, 8]; tp = t[act, 9]
    base = t0.min()
    print(f"{cname:26s} {us:6.1f}us (traced run {h0.elapsed_time(h1)*1000:6.1f}) ctas={int(act.sum())} "
          f"tiles/cta={m[6]:.1f} {s} | start spread {(t0.max()-base)/1e3:.1f}us pdl_pass {(tp.min()-base)/1e3:.1f}.."
          f"{(tp.max()-base)/1e3:.1f} full1 {(t[act,10].min()-base)/1e3:.1f}..{(t[act,10].max()-base)/1e3:.1f} acc1 {(t[act,11].min()-base)/1e3:.1f}..{(t[act,11].max()-base)/1e3:.1f} end {(t1.min()-base)/1e3:.1f}..{(t1.max()-base)/1e3:.1f}us", flush=True)
