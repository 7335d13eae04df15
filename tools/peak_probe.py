"""Print the measured butterfly ceilings (edl_bfly_peak) of every prime of the C1 chain."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_13638_b200 import edl

ctx = edl.Context(edl.params_from_depth(4))
print(json.dumps({"lib": os.environ.get("EDL_LIB", "default"),
                  "Gbfly_s": [round(ctx.bfly_peak(i) / 1e9, 1) for i in range(6)]}))
