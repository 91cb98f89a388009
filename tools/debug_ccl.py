"""Debug helper: GPU RoIs vs oracle extract_rois on the GPU's own cells."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle as O
from paper_2404_09267_b200 import api as A
from tests._helpers import GpuRun
ctx = A.Context(0)
run = GpuRun(ctx, 3840, 2160, 300, seed=1000, keep_mask=False)
gpu = run.run()
cells = run.pipe.cells(300)
bad = 0
for i in range(300):
    want = O.extract_rois(cells[i])
    got = [tuple(r) for r in gpu["rois"][i, :gpu["n_rois"][i]].tolist()]
    if got != want:
        bad += 1
        if bad <= 3:
            print("frame", i, "gpu", len(got), "orc", len(want), flush=True)
            print("  gpu-only", sorted(set(got) - set(want))[:5], " orc-only", sorted(set(want) - set(got))[:5])
            np.save(f"gpurun_out/cells_bad_{i}.npy", cells[i])
print("bad frames", bad)
