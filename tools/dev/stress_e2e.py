"""Dev stress: rebuild the whole C4 mesh every iteration (H2D'd inputs kept on
device), a few sweeps, no synchronisation between phases; reports the first
failure.  usage: python tools/dev/stress_e2e.py ITER SWEEPS [sync]"""
import sys, time, torch
sys.path.insert(0, '.')
import meshgen, paper_1606_00803_b200 as lms
it, sw = int(sys.argv[1]), int(sys.argv[2])
sync = len(sys.argv) > 3 and sys.argv[3] == "sync"
m = meshgen.make_config("C4")
c = [torch.from_numpy(a).cuda() for a in m["coords"]]; e = torch.from_numpy(m["elems"]).cuda()
t = time.time()
k = -1
try:
    for k in range(it):
        g = lms.Mesh.build_csr(c, e)
        g.permute(g.order("original", 0))
        if sync:
            torch.cuda.synchronize()
        g.set_schedule("auto", 0, 0)
        g.smooth(sw)
        out = g.coords()
        torch.cuda.synchronize()
        g.close()
    print("ok", it, "iterations", round(time.time() - t, 1), "s", flush=True)
except Exception as ex:
    print("FAILED at", k, type(ex).__name__, str(ex)[:160], flush=True)
