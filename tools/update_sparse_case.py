"""One fused meta update configuration for ncu: n = 83.9M fp32, projection
max(p, 0); argv[1] = 'sparse' zeroes 3/4 of the gradient samples."""
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
from update_size_probe import run  # noqa: E402

run(83886080, 0.0, len(sys.argv) > 1 and sys.argv[1] == "sparse", steps=3)
