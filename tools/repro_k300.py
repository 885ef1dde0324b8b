import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2112_02179_b200 as P
from tests import _golden
data, g = _golden.load(sys.argv[1] if len(sys.argv) > 1 else "kmeans_k300_wide")
idx = P.deserialize(data, device=0)
print("format", idx.info.format, idx.info.center_bits, idx.info.scale_bits, idx.info.words_per_point)
for B in (1, 6):
    out = P.score_all_batch(idx, g["queries"][:B])
    print(B, "score_all ok", (out[:B] == g["scores"][:B]).all())
