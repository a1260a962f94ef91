import sys, time, torch
sys.path.insert(0, '.')
import meshgen, paper_1606_00803_b200 as lms
mode = sys.argv[1]
m = meshgen.make_config("C4")
c = [torch.from_numpy(a).cuda() for a in m["coords"]]; e = torch.from_numpy(m["elems"]).cuda()
g = lms.Mesh.build_csr(c, e)
g.permute(g.order("original", 0))
t = time.time()
try:
    if mode == "sweeps":
        for k in range(60):
            g.smooth(50)
        torch.cuda.synchronize()
        print("sweeps ok: 3000 launches", round(time.time() - t, 1), "s", flush=True)
    else:
        for k in range(60):
            g.set_schedule("auto", 0, 0)
            g.smooth(5)
        torch.cuda.synchronize()
        print("rebuilds ok: 60 builds", round(time.time() - t, 1), "s", flush=True)
except Exception as ex:
    print("FAILED at", k, type(ex).__name__, str(ex)[:200], flush=True)
