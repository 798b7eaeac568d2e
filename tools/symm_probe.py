"""Probe: torch symmetric memory + multicast (NVLS) availability on this box (torchrun)."""
import json
import os

import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm_mem

local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
out = {"rank": dist.get_rank()}
try:
    t = symm_mem.empty(1 << 20, dtype=torch.uint8, device="cuda")
    h = symm_mem.rendezvous(t, dist.group.WORLD.group_name)
    out.update(backend=str(symm_mem.get_backend(torch.device("cuda"))), mc_ptr=int(h.multicast_ptr),
               nptr=len(h.buffer_ptrs), buf_ptr=int(h.buffer_ptrs[dist.get_rank()]), t_ptr=t.data_ptr())
except Exception as e:
    out["error"] = repr(e)[:300]
print(json.dumps(out), flush=True)
dist.destroy_process_group()
