import os, torch, torch.distributed as dist
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29561")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
import torch.distributed._symmetric_memory as symm
t = symm.empty((1024,), dtype=torch.float32, device="cuda")
h = symm.rendezvous(t, dist.group.WORLD.group_name)
print("rank", h.rank, "world", h.world_size)
print("buffer_ptrs", h.buffer_ptrs, "t.data_ptr", t.data_ptr())
print("signal_pad_ptrs", h.signal_pad_ptrs, "signal_pad_size", getattr(h, "signal_pad_size", None))
print([n for n in dir(h) if not n.startswith("_")])
dist.destroy_process_group()
