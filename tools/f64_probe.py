import sys
sys.path.insert(0, "."); sys.path.insert(0, "tools")
import torch
from paper_1606_05696_b200 import _lib
from tc_probe import run
print("probe DMMA TF/s", round(_lib.probe_fp64_peak("dmma"), 2), "DFMA TF/s", round(_lib.probe_fp64_peak("dfma"), 2))
for (m, n, k, P) in ((128, 128, 32, 1), (200, 72, 100, 3), (256, 256, 256, 4), (66, 130, 34, 2)):
    for opa in "NT":
        for opb in "NT":
            kern, err, _ = run(opa, opb, m, n, k, P, dtype=torch.float64, which="tensor")
            print(f"{m}x{n}x{k} P={P} {opa}{opb} {kern} err={err:.2e}", flush=True)
for (m, n, k, P) in ((256, 256, 256, 256), (512, 512, 512, 64), (1024, 1024, 1024, 8)):
    kern, err, t = run("N", "N", m, n, k, P, dtype=torch.float64, reps=5)
    print(f"{m}x{n}x{k} x{P} NN {kern} err={err:.2e} {t:.3f} ms {2*m*n*k*P/t/1e9:.2f} TF/s", flush=True)
