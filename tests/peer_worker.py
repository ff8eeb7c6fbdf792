"""Worker for tests/test_peer_gpu.py (launched by torch.distributed.run, one
process per GPU): trains the config-1 golden case through comm_step with the
peer-store exchange (torch symmetric memory buffers, isg_route_pack_peer,
isg_band_fold_peer, signal-pad barriers) and with point-to-point NCCL copies,
densify included, and checks both against the single-GPU engine bit for bit.
Rank 0 writes the verdict as JSON to argv[1]."""

from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main(out_path: str) -> None:
    import paper_2509_05216_b200 as P
    from paper_2509_05216_b200 import distributed as D
    from paper_2509_05216_b200.engine import Trainer
    from golden_io import cam_from, load
    from oracle import train as T
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    world, rank = dist.get_world_size(), dist.get_rank()
    d = load("config1")
    cams = []
    for i in range(d["images_u8"].shape[0]):
        c = cam_from(d, prefix=f"cam{i}_")
        cams.append(P.Camera(c.rotation, c.translation, c.fx, c.fy, c.cx, c.cy, c.width, c.height))
    gt = torch.from_numpy(d["images_u8"]).to(dev)
    ext = T.scene_extent(cams)
    iters = 6
    cfg = P.TrainConfig(iterations=iters, densify_start=2, densify_interval=2, densify_stop=5)
    cloud = P.cloud_from_points(d["points"], d["init_log_scales"], device=dev)
    sched = P.build_schedule(iters, len(cams), 0)
    tr = Trainer(cloud.copy(), cams[0].width, cams[0].height, cfg, ext, dev,
                 canon_rows=D.CANON_ROWS)
    for it in range(1, iters + 1):
        tr.step(it, cams[sched[it - 1]], gt[sched[it - 1]])
        if tr.densify_due(it):
            tr.densify(it)
    ref_losses = tr.loss_dev[1:iters + 1].tolist()
    ref = tr.cloud
    result = {"world": world}
    for mode in ("peer", "nccl"):
        comm = D.TorchComm(peers=mode == "peer", height=cams[0].height, width=cams[0].width,
                           device=dev)
        (rs,), smap, part = D.make_ranks(cloud.copy(), cams[0].width, cams[0].height, cfg, ext,
                                         world, dev, only_rank=rank)
        losses = []
        for it in range(1, iters + 1):
            losses.append(float(D.comm_step(rs, comm, cams[sched[it - 1]], gt[sched[it - 1]],
                                             it)[0]))
            if D.densify_due(cfg, it):
                rs = D.comm_densify(rs, comm, it)
                smap = D.partition_gaussians(sum(D._all_sizes(rs, comm)), world)
        full = {}
        for k in P.PARAM_NAMES:
            t = getattr(rs.cloud, k).contiguous()
            bufs = [torch.empty((smap.sizes[w],) + tuple(t.shape[1:]), dtype=t.dtype, device=dev)
                    for w in range(world)]
            dist.all_gather(bufs, t)
            full[k] = torch.cat(bufs, 0)
        result[mode] = {
            "losses_equal": losses == ref_losses,
            "params_equal": all(torch.equal(full[k], getattr(ref, k)) for k in P.PARAM_NAMES),
            "count": int(full["positions"].shape[0]), "ref_count": ref.count,
            "peer_capacity": [comm.peers.cap_r, comm.peers.cap_g] if comm.peers else None,
        }
    if rank == 0:
        with open(out_path, "w") as f:
            json.dump(result, f)
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1])
