"""Run 3 rounds of a K=4 (K=8 / K=36 variants) federation at world = WORLD_SIZE with per-round
evaluation; rank 0 saves theta | velocity | eval ppls (npy) and the runner's
resume directory (<out>.ckpt/: checkpoint.phck, velocity.phck, state.json)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2411_02908_b200 import fedsim as F  # noqa: E402

out, server = sys.argv[1], sys.argv[2]
world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
local = int(os.environ.get("LOCAL_RANK", "0"))
nccl_id = None
if world > 1:
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    obj = [F.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    nccl_id = obj[0]
cfg = F.ModelConfig(1, 32, 2, 4, 64, 16)
theta0 = F.TransformerModel(cfg).init_params(1)
local_cfg = F.LocalTrainConfig(model=cfg, schedule=F.LrSchedule(2e-3, 16, 160, 0.1),
                               local_steps=4, batch_size=4)
srv = F.ServerOptConfig() if server == "fedavg" else F.diloco_server_opt()
drop = server.endswith("_drop")  # parameter server with a simulated dropout in round 1
# diloco_k8: 8 of 12 clients per round (2 local clients per rank on 4 GPUs: the
# KM = 8 peer kernel).  diloco_many: 36 of 40 with 20 dropped in round 1, so one
# rank holds more local models than the peer path takes: every rank
# must agree on the NCCL path.
POP, K = {"diloco_k8": (12, 8), "diloco_many": (40, 36)}.get(server, (6, 4))
plan = F.partition_iid(F.generate_corpus("web", 10000 * POP, 7, 64), POP, 16, 7)
if server == "central":  # DDP baseline: 6 workers, per-step gradient all-reduce
    ccfg = F.CentralizedConfig(model=cfg, schedule=F.LrSchedule(2e-3, 16, 160, 0.1), n_workers=6,
                               global_batch=12, total_steps=4, opt_reset_interval=2)
    res = F.run_centralized(ccfg, plan, 42, theta0, device=local, precision="f32", rank=rank,
                            world=world, nccl_id=nccl_id)
    if rank == 0:
        np.save(out, np.concatenate([res.theta, [s.loss for s in res.steps], res.cursors]))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    sys.exit(0)
es = F.EvalSet(["web"], 40, 7, cfg, 8)  # 5 batches: uneven over 2 or 4 ranks
many = server == "diloco_many"
topo = F.Topology.kParameterServer if (drop or many) else F.Topology.kRingAllReduce
# with a dropout: the second sampled client of round 1 never reports (3 survivors)
dropouts = [(1, F.sample_clients(6, 4, 42, 1)[1])] if drop else []
if many:
    dropouts = [(1, c) for c in F.sample_clients(POP, K, 42, 1)[1::2][:18]] + \
               [(1, F.sample_clients(POP, K, 42, 1)[0]), (1, F.sample_clients(POP, K, 42, 1)[2])]
runner = F.FederationRunner(F.FederationConfig(POP, K, 3, topo, 42), local_cfg,
                            srv, plan, theta0, device=local, precision="f32", rank=rank,
                            world=world, nccl_id=nccl_id, eval_set=es, eval_every=1,
                            dropouts=dropouts)
ppls = [runner.run_round().eval_ppl for _ in range(3)]
theta = runner.theta()
vel = runner.velocity()
ckpt = out + ".ckpt"
if rank == 0:
    os.makedirs(ckpt, exist_ok=True)
if world > 1:
    dist.barrier()
runner.save(ckpt)
if rank == 0:
    np.save(out, np.concatenate([theta, vel, np.array(ppls)]))
if world > 1:
    dist.barrier()
    dist.destroy_process_group()
