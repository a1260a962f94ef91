#!/usr/bin/env python
"""Dev tool: time lms_smooth on one config under several schedules / tiles /
lags / orderings (CUDA events, warm), one JSON line per variant."""
import argparse
import itertools
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import meshgen  # noqa: E402
import paper_1606_00803_b200 as lms  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="C4")
    p.add_argument("--orderings", default="original")
    p.add_argument("--variants", default="s1:0:0,s3:4096:0")
    p.add_argument("--sweeps", type=int, default=20)
    p.add_argument("--reps", type=int, default=3)
    a = p.parse_args()
    m = meshgen.make_config(a.config)
    coords = [torch.from_numpy(c).cuda() for c in m["coords"]]
    elems = torch.from_numpy(m["elems"]).cuda()
    for ordering in a.orderings.split(","):
        gm = lms.Mesh.build_csr(coords, elems)
        t0 = time.time()
        perm = gm.order(ordering, 803)
        torch.cuda.synchronize()
        t_order = time.time() - t0
        gm.permute(perm)
        base = gm.coords()
        inf = gm.info()
        for var in a.variants.split(","):
            parts = var.split(":")
            kind, tile, lag = parts[:3]
            os.environ["LMS_OPTS"] = parts[3] if len(parts) > 3 else "4"
            for idx, env in ((4, "LMS_S3_CTAS_PER_SM"), (5, "LMS_S3_RING")):
                if len(parts) > idx and parts[idx]:
                    os.environ[env] = parts[idx]
                else:
                    os.environ.pop(env, None)
            gm.set_schedule(kind, int(tile), int(lag), tiling=parts[6] if len(parts) > 6 and parts[6] else "auto")
            gm.import_coords(base)
            gm.smooth(1)
            torch.cuda.synchronize()
            si = gm.schedule_info()
            ts = []
            for _ in range(a.reps):
                e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
                e0.record(); gm.smooth(a.sweeps); e1.record(); torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            t = min(ts) / a.sweeps
            nf = si["n_free"]
            bsw = 4 * (inf["V"] + 1) + 4 * inf["nnz"] + 8 * inf["dim"] * inf["V"] + 8 * inf["dim"] * nf
            print(json.dumps(dict(config=a.config, ordering=ordering, var=var, sched=si, us_per_sweep=t * 1e3,
                                  gvups=nf / (t / 1e3) / 1e9, gbs=bsw / (t / 1e3) / 1e9,
                                  frac=bsw / (t / 1e3) / 1e9 / 6546.2, t_order_s=t_order)), flush=True)
        gm.close()


if __name__ == "__main__":
    main()
