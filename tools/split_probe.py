import sys
sys.path.insert(0, ".")
sys.path.insert(0, "tools")
from tc_probe import run
for (m, n, k, P) in ((128, 128, 256, 8), (256, 256, 1024, 2)):
    for opa, opb in (("T", "N"), ("N", "T")):
        kern, err, t = run(opa, opb, m, n, k, P, which="tensor")
        print(f"{m}x{n}x{k} {opa}{opb} {kern} err={err:.2e}")
