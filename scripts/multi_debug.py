"""Dev repro: lms_min_bracelet_multi on one GPU (host exchange)."""
import sys

sys.path.insert(0, ".")
from paper_1510_01041_b200 import _native, workloads  # noqa: E402
from paper_1510_01041_b200.backend import record_from_native  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
world = int(sys.argv[2]) if len(sys.argv) > 2 else 1
pts = workloads.contaminated_line_points(n, 0)
a, b = pts[:, 0].copy(), pts[:, 1].copy()
q = n // 2 + 1
ctx = _native.Context()
ctx.upload(a, b)
want = record_from_native(ctx.solve(q, 0, n * (n - 1) // 2))
print("single", want, flush=True)
got = record_from_native(_native.min_bracelet_multi(a, b, q, [0] * world))
print("multi", got, got == want, flush=True)
