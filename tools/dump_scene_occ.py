"""Write the bench scene's env occupancy (512^3) to a raw file for tools/phase_timing."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
from paper_2407_02363_b200.engine import MapCycle
d = bench.desk7()
cyc = MapCycle(bench.DIMS, bench.VS, bench.ORIGIN, d["links"], bench.VS, d["o_links"], bench.POINTS, 32)
pts, frames, centers = bench.scene_inputs(0, 0, d)
cyc.step(pts, frames, centers)
env, _, _ = cyc.grids()
occ = env.occupancy_mask().view(np.uint8)
occ.tofile(sys.argv[1])
print("occupied", int(occ.sum()))
