"""One simulated rank of the G-way cfg5 z-slab split (development aid, ncu
target): the slab of 2048/G planes at its global z0, GraphedSlabStages with
fused=False, a few replays.  usage: python tools/prof_rank.py G [rank] [reps]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2012_08099_b200 import distributed as pdist  # noqa: E402
from paper_2012_08099_b200 import engine  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 8
R = int(sys.argv[2]) if len(sys.argv) > 2 else G - 1
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
z0, z1 = pdist.slab_bounds(2048, G, R)
slab = engine.synth_noise(2048, 2048, z0, z1 - z0, 5)
st = engine.GraphedSlabStages(slab, 6, z0=z0, fused=False, n_global=2048)
for _ in range(reps):
    st.replay_project(); st.replay_moments2d(); res = st.replay_derive()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    st.replay_project(); st.replay_moments2d(); res = st.replay_derive()
e1.record()
torch.cuda.synchronize()
print(f"G={G} rank={R} z0={z0} planes={z1 - z0}: {e0.elapsed_time(e1) / 10:.4f} ms per step, status {int(res.status[0])}")
