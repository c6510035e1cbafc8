import os, sys
mode = sys.argv[1]
if mode == "inproc":
    os.environ["NCCL_DEBUG_FILE"] = "/dev/stderr"
elif mode == "none":
    os.environ["NCCL_DEBUG"] = "WARN"
import torch, torch.distributed as dist
r = int(os.environ["LOCAL_RANK"]); torch.cuda.set_device(r)
dist.init_process_group("nccl", device_id=torch.device("cuda", r))
t = torch.ones(1, device="cuda"); dist.all_reduce(t)
if r == 0: print("RESULT", mode, t.item(), flush=True)
dist.destroy_process_group()
