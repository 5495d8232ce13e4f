"""A/B helper: run bench.py with OrderedWire's small-bucket caps overridden
(GS_LL_MAX_ELEMS / GS_SMALL_CAP_ELEMS in the environment), e.g. under torchrun
`tools/ab_small_cap.py --gpus 4 --algorithm ordered --theta 262144`.  Tuning
only; the product constants live in dist.OrderedWire."""
import os
import runpy
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1807_11205_b200.dist import OrderedWire  # noqa: E402

for key in ("LL_MAX_ELEMS", "SMALL_CAP_ELEMS"):
    if os.environ.get("GS_" + key):
        setattr(OrderedWire, key, int(os.environ["GS_" + key]))
sys.argv[0] = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "bench.py")
runpy.run_path(sys.argv[0], run_name="__main__")
