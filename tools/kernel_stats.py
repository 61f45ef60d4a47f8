"""Instrumented ray cast at config 2 (a RO_STATS=1 build, RESOCT_LIB=...):
prints the work counters, including the instrumentation counters 5..7
(probe misses, tap loads, full TF evaluations), per orbit pose."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2309_04393_b200 import scenarios  # noqa: E402
from paper_2309_04393_b200.camera import orbit_path  # noqa: E402
from paper_2309_04393_b200.render import MODE_RESIDENCY, FramePass  # noqa: E402

scn = scenarios.cycif(device="cuda")
eng = scenarios.build_engine(scn)
rows = []
for i, cam in enumerate(orbit_path(int(sys.argv[1]) if len(sys.argv) > 1 else 4)):
    fp = FramePass(MODE_RESIDENCY, eng.paging, eng.octree, scn.channels, cam, scn.render)
    fp.render()
    fp.collect()
    torch.cuda.synchronize()
    c = fp.buf.counters.cpu().tolist()
    h = fp.buf.hist.cpu().numpy()
    rows.append({"pose": i, "steps": c[0], "evaluated": c[1], "skipped": c[2],
                 "misses": c[5], "tap_loads": c[6], "tf_evals": c[7],
                 "fetches": int(h.sum()), "hist": h.tolist()})
    print(json.dumps(rows[-1]), flush=True)
