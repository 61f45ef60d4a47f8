"""Device-side split of render_frame()'s frame at config 2: the same launch
sequence as render._run with CUDA events between the stages, the image /
per-pixel counts stored into pinned host memory (zero-copy) or into device
memory (the bench's device path)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_04393_b200 import _native as N, render as R, scenarios  # noqa: E402
from paper_2309_04393_b200.camera import orbit_path  # noqa: E402


def main():
    scn = scenarios.cycif(device="cuda")
    eng = scenarios.build_engine(scn)
    cams = orbit_path(20)
    res = {}
    for zero_copy in (True, False, True):
        st = {"render": [], "collect": [], "copies": []}
        for i, c in enumerate(cams):
            fp = R.FramePass(R.MODE_RESIDENCY, eng.paging, eng.octree, scn.channels, c,
                             scn.render)
            buf = fp.buf
            shapes = R._result_shapes(buf)
            (img, pixr, req, small), owned = R._RESULTS.acquire(shapes)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            ev[0].record()
            if zero_copy:
                fp.render(N.Outputs(img.data_ptr(), buf.required.data_ptr(), pixr.data_ptr(),
                                    buf.hist.data_ptr(), buf.counters.data_ptr()))
            else:
                fp.render()
            ev[1].record()
            fp.collect(asynchronous=True)
            ev[2].record()
            req.copy_(buf.required, non_blocking=True)
            small.copy_(buf.small, non_blocking=True)
            ev[3].record()
            torch.cuda.synchronize()
            if owned:
                R._RESULTS.handout(shapes, (img, pixr, req, small), (img, pixr, req))
            st["render"].append(ev[0].elapsed_time(ev[1]))
            st["collect"].append(ev[1].elapsed_time(ev[2]))
            st["copies"].append(ev[2].elapsed_time(ev[3]))
        res["zero_copy" if zero_copy else "device"] = {k: sum(v) / len(v) for k, v in st.items()}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
