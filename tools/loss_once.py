"""One 1080p cs_training_loss call (K13) for ncu captures."""
import torch

from paper_2404_01133_b200 import _lib, device

H, W = 1080, 1920
g = torch.Generator(device="cuda").manual_seed(1)
img = torch.rand((H, W, 3), generator=g, device="cuda")
ref = (img + 0.1 * torch.randn((H, W, 3), generator=g, device="cuda")).clamp(0, 1)
loss = torch.zeros(1, dtype=torch.float64, device="cuda")
grad = torch.empty_like(img)
for _ in range(3):
    _lib.check(_lib.load().cs_training_loss(device.context(0), img.data_ptr(), ref.data_ptr(), H, W, 0.2,
                                            loss.data_ptr(), grad.data_ptr(), device.stream_handle()))
torch.cuda.synchronize()
print("loss", float(loss))
