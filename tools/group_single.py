"""One grouped execute_plans call over the 28 plain (or 8 exceptional) cases
of the n=256 sweep (for ncu).  argv: [plain|bb] [n] [reps]"""
import sys
import torch
sys.path.insert(0, ".")
import paper_1606_05696_b200 as sbt
which = sys.argv[1] if len(sys.argv) > 1 else "plain"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
EXC = {"3.4", "3.6", "4.4", "4.6", "5.4", "5.6", "6.4", "6.6"}
a2 = torch.rand(n * n, device="cuda") * 2 - 1
b3 = torch.rand(n ** 3, device="cuda") * 2 - 1
calls = []
for case in sbt.enumerate_cases(2, 3):
    if (case.case_id in EXC) != (which == "bb"):
        continue
    spec = sbt.ContractionSpec(case.labels_a, case.labels_b, case.labels_c)
    lays = [sbt.Layout.packed([n] * len(l)) for l in (spec.labels_a, spec.labels_b, spec.labels_c)]
    a = sbt.DenseTensor(lays[0], a2 if lays[0].size == n * n else b3)
    b = sbt.DenseTensor(lays[1], a2 if lays[1].size == n * n else b3)
    c = sbt.DenseTensor(lays[2], torch.empty(n ** 3, device="cuda"))
    calls.append((sbt.plan_single_mode(spec, *lays), a, b, 1.0, 0.0, c))
for _ in range(reps):
    sbt.execute_plans(calls)
torch.cuda.synchronize()
print(which, len(calls), "cases")
