import sys, torch, numpy as np
sys.path.insert(0, '.')
import bench
from paper_2509_05216_b200 import synthetic as S
import paper_2509_05216_b200 as P
from paper_2509_05216_b200.engine import Trainer
from paper_2509_05216_b200.training import TrainConfig, TrainDataset, PointCloud
name = sys.argv[1]
dev = torch.device("cuda", 0)
nv = S.CONFIGS[name][4]
wl = S.make_workload(name, dev, view_ids=[0, 1])
ext = TrainDataset(wl.cameras, np.zeros((nv, 1, 1, 3)), PointCloud(wl.points, wl.normals)).scene_extent
tr = Trainer(P.cloud_from_points(wl.points, wl.log_scales, 1, dev), wl.resolution, wl.resolution, TrainConfig(iterations=3, densify=False), ext, dev)
print(bench.api_render_timing(tr, wl, 0, torch.float32), flush=True)
print(bench.api_render_timing(tr, wl, 0, torch.float64), flush=True)
