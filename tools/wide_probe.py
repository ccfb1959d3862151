"""Which kernel runs a strided-basis block update (GMRES W -= V H) at each width kp."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2504_02117_b200 as bk  # noqa: E402

ctx = bk.Context(0)
n, k, ldv = int(sys.argv[1]) if len(sys.argv) > 1 else 2097152, 12, 780
V = torch.randn(n, ldv, dtype=torch.float64, device="cuda")
W = torch.randn(n, k, dtype=torch.float64, device="cuda")
for kp in [216, 228, 240, 252, 264, 456, 468, 516, 576]:
    H = torch.randn(kp, k, dtype=torch.float64, device="cuda")
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        bk.block_update(ctx, W, V[:, :kp], H, a=1.0, s=-1.0)
        torch.cuda.synchronize()
    names = [e.name for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    import re; print(kp, [re.sub(r"\(.*", "", nm.replace("(anonymous namespace)", "")) for nm in names])
