"""Run one of the 36 cases a few times (for ncu). argv: case_id n [f32|f64] [reps]"""
import sys
import torch
sys.path.insert(0, ".")
import paper_1606_05696_b200 as sbt
from paper_1606_05696_b200 import _lib
cid, n = sys.argv[1], int(sys.argv[2])
dtype = torch.float64 if (len(sys.argv) > 3 and sys.argv[3] == "f64") else torch.float32
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
case = sbt.find_case(2, 3, cid)
spec = sbt.ContractionSpec(case.labels_a, case.labels_b, case.labels_c)
lays = [sbt.Layout.packed([n] * len(l)) for l in (spec.labels_a, spec.labels_b, spec.labels_c)]
a = sbt.DenseTensor(lays[0], torch.rand(lays[0].size, device="cuda", dtype=dtype))
b = sbt.DenseTensor(lays[1], torch.rand(lays[1].size, device="cuda", dtype=dtype))
c = sbt.DenseTensor(lays[2], torch.empty(lays[2].size, device="cuda", dtype=dtype))
plan = sbt.plan_single_mode(spec, *lays)
for _ in range(reps):
    sbt.execute_plan(plan, a, b, 1.0, 0.0, c)
torch.cuda.synchronize()
print(cid, n, dtype, _lib.last_kernel())
