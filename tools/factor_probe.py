"""Run the HOOI factor update (sbt_hooi_factor_f32) on a 512 x 32 x 32 partial
core in each mode, plus the acc64 core product: a small target for ncu."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_1606_05696_b200 import tucker as tk
from paper_1606_05696_b200.layout import DenseTensor
rng = np.random.default_rng(0)
for dims, mode in (((512, 32, 32), 0), ((32, 512, 32), 1), ((32, 32, 512), 2)):
    t = DenseTensor.from_array(rng.standard_normal(dims), dtype="float32")
    warm = torch.linalg.qr(torch.randn(512, 32, dtype=torch.float64, device="cuda"))[0]
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    for _ in range(3):
        tk._factor_device(t, mode, 32, warm, st, 0)
    if mode == 2:
        for _ in range(3):
            tk._mode_product_acc64(t, warm, 2)
torch.cuda.synchronize()
print("ok")
