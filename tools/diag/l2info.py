import torch
p = torch.cuda.get_device_properties(0)
print(p.name, "L2", p.L2_cache_size, "persist max", getattr(p, "persisting_l2_cache_max_size", None))
import ctypes
cu = ctypes.CDLL("libcudart.so")
