"""One captured config-5 formation pass replayed inside a profiler range
(for `ncu --profile-from-start off`) -- development aid."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2101_08053_b200 import cases as C
from paper_2101_08053_b200.assembly import GraphFormation, form
nel = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
eager = "eager" in sys.argv
c5 = C.baseline_config(5, nel=nel)
b2d, cfg = C.build_space(None, nel, 4, curves=c5["curves"])
if "stamps" in sys.argv:
    from paper_2101_08053_b200 import _lib as L, assembly as A
    world = int(sys.argv[sys.argv.index("world") + 1]) if "world" in sys.argv else 1
    K = cfg.active_index()[0]["K"]
    rr = (0, K // world)
    gf = GraphFormation(b2d, cfg, None, "dwq", row_range=rr)     # plans warmed
    del gf
    A.STAMPS = L.Stamps()
    gf = GraphFormation(b2d, cfg, None, "dwq", row_range=rr)
    # the capture pass is the last set of stamps recorded
    names = A.STAMPS.names
    k = len(names) - 1 - names[::-1].index("start")
    for _ in range(5):
        gf.run()
    torch.cuda.synchronize()
    t = A.STAMPS.buf.cpu().numpy()
    base = int(t[k])
    for i in range(k, len(names)):
        print(f"{names[i]:16s} {(int(t[i]) - base) / 1e3:8.1f} us")
    cut = gf.f._setup.cut
    gp = cut["grp_pts"].cpu().numpy()
    import numpy as np
    n = np.diff(gp)
    print("ngroups", cut["ngroups"], "npts", cut["npts"], "pts/group mean", n.mean(), "max", n.max(),
          "pcts", np.percentile(n, [10, 50, 90, 99]), "cut elements", cut["grp_ptr"].numel() - 1,
          "nraw", gf.f._ndesc, "nint", gf.f._nint)
    sys.exit(0)
if eager:
    # the capture-mode schedule run eagerly (ncu cannot replay the graph's nodes)
    _, csr = form(b2d, cfg, None, "dwq")
    cap = {"nnz": csr.nnz}
    for _ in range(3):
        form(b2d, cfg, None, "dwq", capture=cap)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    form(b2d, cfg, None, "dwq", capture=cap)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
else:
    gf = GraphFormation(b2d, cfg, None, "dwq")
    for _ in range(3):
        gf.run()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    gf.run()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print("launches_per_pass", gf.launches_per_pass, "nnz", gf.nnz)
