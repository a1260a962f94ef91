#!/usr/bin/env python
"""Soak test of the end-to-end path (a race detector, not a benchmark).

Runs the bench's e2e job -- lms_build_csr_host -> lms_order -> lms_permute ->
lms_smooth(S) -> coordinates -- many times with N jobs in flight on N streams
and compares every job's coordinates, bit for bit, with the first job's of
the same ordering (whose parity against the oracle is the test suite's job:
tests/test_gpu_fullsize.py).  The sweeps are deterministic (colour-GS, Eq. 1
P:244-251 in neighbour order), so any difference, any watchdog error or any
CUDA error is a race in the schedule build or the sweep kernel.

  python tools/soak.py --config C4 --orderings original:600,bfs:60,random:40
"""
import argparse
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import meshgen  # noqa: E402
import paper_1606_00803_b200 as lms  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--orderings", default="original:600,bfs:60,random:40")
    ap.add_argument("--sweeps", type=int, default=50)
    ap.add_argument("--jobs-in-flight", type=int, default=4)
    ap.add_argument("--batch", type=int, default=8)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    m = meshgen.make_config(args.config)
    dim = m["dim"]
    hc = [torch.from_numpy(c).pin_memory() for c in m["coords"]]
    he = torch.from_numpy(m["elems"]).pin_memory()
    nj = args.jobs_in_flight
    strs = [torch.cuda.Stream() for _ in range(nj)]
    report = {"config": args.config, "sweeps": args.sweeps, "jobs_in_flight": nj, "orderings": {}}
    ok = True
    for spec in args.orderings.split(","):
        kind, n = spec.split(":")
        n = int(n)
        seed = meshgen.RANDOM_ORDER_SEED if kind == "random" else 0
        ref = None
        done = bad = 0
        t0 = time.time()
        while done < n:
            keep = []
            for k in range(min(args.batch, n - done)):
                with torch.cuda.stream(strs[k % nj]):
                    g = lms.Mesh.build_csr_host(hc, he)
                    g.set_async_errors(True)
                    p = g.order(kind, seed)
                    g.permute(p)
                    g.smooth(args.sweeps)
                    keep.append((g, g.coords(), p))
            torch.cuda.synchronize()
            for g, out, p in keep:
                g.check()  # raises on a watchdog / CUDA error
                if ref is None:
                    ref = [o.clone() for o in out] + [p.clone()]
                else:
                    same = all(torch.equal(o.view(torch.int64), r.view(torch.int64)) for o, r in zip(out, ref[:dim]))
                    same = same and torch.equal(p, ref[dim])
                    bad += 0 if same else 1
                g.close()
                done += 1
        dt = time.time() - t0
        report["orderings"][kind] = {"jobs": done, "sweep_launches": done * args.sweeps, "mismatches": bad,
                                     "wall_s": round(dt, 1)}
        print(json.dumps({kind: report["orderings"][kind]}), flush=True)
        ok = ok and bad == 0
    report["ok"] = ok
    print("SOAK " + ("OK " if ok else "FAILED ") + json.dumps(report), flush=True)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
