import torch
print("peer", torch.cuda.can_device_access_peer(0, 1), torch.cuda.can_device_access_peer(1, 0))
