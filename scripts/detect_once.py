"""Dev: detect_lines on the config-5 image, a few times (for ncu)."""
import sys

sys.path.insert(0, ".")
import paper_1510_01041_b200 as lms  # noqa: E402
from paper_1510_01041_b200 import workloads  # noqa: E402

img = workloads.config5_image(0)
p = lms.HoughParams.for_image(4096, 4096, 20.0, 20.0)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    d = lms.detect_lines(img, p, "lms", 64)
print(len(d))
