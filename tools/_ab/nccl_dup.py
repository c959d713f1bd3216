import os, torch, torch.distributed as dist
dist.init_process_group("nccl")
r = dist.get_rank()
torch.cuda.set_device(0)
x = torch.full((4,), float(r), device="cuda")
if r == 0:
    dist.send(x, 1)
else:
    dist.recv(x, 0)
torch.cuda.synchronize()
print("rank", r, x.tolist(), flush=True)
dist.destroy_process_group()
