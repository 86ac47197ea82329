import sys, os
sys.path.insert(0, os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "tests"))
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import test_gpu_fuzz as t
from test_gpu_parity import run_parity
geo, n, spec, mode, wo = t._case(82)
B = geo[3]
nb = 2 * sum(-(-x[0] // B) for x in spec) + 64
variant = sys.argv[1] if len(sys.argv) > 1 else "orig"
if variant == "one":
    mode = "one"
if variant == "wo0":
    wo = 0
run_parity(geo, [nb] * n, spec, seed=82, per_gpu_launch=mode == "per_gpu", a2a=mode == "a2a", work_order=wo, degrees=(2, 4, 8, 16))
print("ok", variant)
