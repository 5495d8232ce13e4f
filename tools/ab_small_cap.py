"""A/B helper: run bench.py (or, with GS_AB_SCRIPT, another script such as
tools/allreduce_sweep.py) with OrderedWire's size constants overridden from
the environment (GS_LL_MAX_ELEMS, GS_SMALL_CAP_ELEMS, GS_MIN_ELEMS_PER_CTA,
GS_PUSH_MAX_BYTES),
e.g. under torchrun `tools/ab_small_cap.py --gpus 4 --algorithm ordered
--theta 262144`.  Tuning only; the product constants live in dist.OrderedWire."""
import os
import runpy
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1807_11205_b200.dist import OrderedWire  # noqa: E402

for key in ("LL_MAX_ELEMS", "SMALL_CAP_ELEMS", "MIN_ELEMS_PER_CTA", "PUSH_MAX_BYTES"):
    if os.environ.get("GS_" + key):
        setattr(OrderedWire, key, int(os.environ["GS_" + key]))
sys.argv[0] = os.path.join(ROOT, os.environ.get("GS_AB_SCRIPT", "bench.py"))
runpy.run_path(sys.argv[0], run_name="__main__")
