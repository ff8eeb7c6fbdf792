import sys, torch, numpy as np
sys.path.insert(0, '.')
import paper_2509_05216_b200 as P
from paper_2509_05216_b200 import synthetic as S
from paper_2509_05216_b200.engine import Trainer
from paper_2509_05216_b200.training import TrainConfig, TrainDataset, PointCloud, build_schedule
dev = torch.device("cuda", 0)
name = sys.argv[1]
nv = S.CONFIGS[name][4]
sched = build_schedule(3, nv, 0)
wl = S.make_workload(name, dev, view_ids=sched)
ext = TrainDataset(wl.cameras, np.zeros((nv, 1, 1, 3)), PointCloud(wl.points, wl.normals)).scene_extent
cfg = TrainConfig(iterations=3, densify=False, eval_interval=0)
tr = Trainer(P.cloud_from_points(wl.points, wl.log_scales, 1, dev), wl.resolution, wl.resolution, cfg, ext, dev)
tr.r.chunk = 0
tr.step(1, wl.cameras[sched[0]], wl.images_u8[0])
torch.cuda.synchronize()
r = tr.r
off = r.offsets.cpu().numpy().astype(np.int64)
cm = r.cmask.cpu().numpy().view(np.uint32)
res = wl.resolution; txn = res // 16
nlast = r.n_last.cpu().numpy().reshape(res, res)
both = either = 0; work_half = 0; lens=[]
for tl in range(len(off) - 1):
    e0, n = off[tl], off[tl + 1] - off[tl]
    ty, tx = divmod(tl, txn)
    blk = nlast[ty*16:(ty+1)*16, tx*16:(tx+1)*16]
    wq = [blk[0:8, 0:8].max(), blk[0:8, 8:16].max(), blk[8:16, 0:8].max(), blk[8:16, 8:16].max()]
    for b in range((n + 31) // 32):
        base = 4 * ((e0 >> 5) + tl + b)
        w = [cm[base + q] if b * 32 < wq[q] else 0 for q in range(4)]
        top = int(w[0] | w[1]); bot = int(w[2] | w[3])
        both += bin(top & bot).count("1"); either += bin(top | bot).count("1")
        work_half += bin(top).count("1") + bin(bot).count("1")
print(name, "either", either, "both", both, "f2", both / either, "half-walks per entry", work_half / either)
