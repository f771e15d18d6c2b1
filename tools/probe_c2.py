"""Phase probes of the C2 small-core kernels (RSVD_PROBE_FQ=1): per-pass
cycle counts of the fused CholeskyQR and the Jacobi sweep count."""
import os
import sys

os.environ["RSVD_PROBE_FQ"] = "1"
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2402_17794_b200 as eng  # noqa: E402

cfg = bench.CONFIGS["C2"]
a = bench.make_input(cfg, torch.device("cuda", 0))
for _ in range(3):
    eng.rsvd(a, eng.SketchConfig(20, 5, 2, eng.RangeMode.power, 1))
torch.cuda.synchronize()
