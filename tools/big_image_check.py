"""Three training steps at an image of more than 65536 tiles (4-byte tile
keys), e.g. 8192^2: the step runs and its loss is finite and decreasing-ish."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_2509_05216_b200 as P
from paper_2509_05216_b200 import synthetic as S
from paper_2509_05216_b200.engine import Trainer
from paper_2509_05216_b200.training import TrainConfig, TrainDataset, PointCloud, build_schedule

res = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
dev = torch.device("cuda", 0)
nv = S.CONFIGS["config2"][4]
sched = build_schedule(3, nv, 0)
wl = S.make_workload("config2", dev, view_ids=sched, resolution=res)
ext = TrainDataset(wl.cameras, np.zeros((nv, 1, 1, 3)), PointCloud(wl.points, wl.normals)).scene_extent
tr = Trainer(P.cloud_from_points(wl.points, wl.log_scales, 1, dev), res, res,
             TrainConfig(iterations=3, densify=False), ext, dev)
for it in range(1, 4):
    tr.step(it, wl.cameras[sched[it - 1]], wl.images_u8[it - 1])
torch.cuda.synchronize()
print("tiles", tr.r.n_tiles, "losses", tr.loss_dev[1:4].tolist(), "E", int(tr.r.offsets[-1]))
assert tr.r.n_tiles > 65536 and all(np.isfinite(tr.loss_dev[1:4].cpu().numpy()))
