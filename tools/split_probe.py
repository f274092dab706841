"""3xTF32 error and speed vs K with/without the split small-term accumulator."""
import os, sys
sys.path.insert(0, ".")
from tools.tc_probe import run
for (m, n, k, P) in ((512, 512, 512, 64), (1024, 1024, 1024, 16), (1024, 1024, 2048, 8), (512, 512, 4096, 8)):
    kern, err, t = run("N", "N", m, n, k, P, reps=5)
    print(f"split={os.environ.get('SBT_TC_SPLITACC','auto')} {m}x{n}x{k} x{P} {kern} err={err:.2e} {t:.3f} ms {2*m*n*k*P/t/1e9:.1f} TF/s", flush=True)
