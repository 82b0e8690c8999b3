import os, sys, torch, torch.distributed as dist
rank = int(os.environ["RANK"]); world = int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda:0"))
t = torch.ones(4, device="cuda:0") * (rank + 1)
try:
    dist.all_reduce(t)
    torch.cuda.synchronize()
    print("rank", rank, "all_reduce ok", t.tolist(), flush=True)
except Exception as e:
    print("rank", rank, "failed:", type(e).__name__, str(e)[:300], flush=True)
dist.destroy_process_group()
