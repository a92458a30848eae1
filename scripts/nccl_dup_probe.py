"""Probe: can two ranks share one GPU in an NCCL communicator (torch.distributed)?"""
import os, torch, torch.distributed as dist
rank = int(os.environ["RANK"]); world = int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
x = torch.full((4,), float(rank + 1), device="cuda")
dist.all_reduce(x)
print("rank", rank, "allreduce ok", x.tolist(), flush=True)
dist.destroy_process_group()
