import os, sys, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests import test_gpu_decode as T
fails = 0
for i in range(int(os.environ.get("N", 12))):
    for name in ("test_decode_layer_matches_oracle_chain", "test_graph_step_with_overlap_matches_oracle_chain"):
        try:
            if name.startswith("test_decode"):
                T.test_decode_layer_matches_oracle_chain(8192, 0.25)
            else:
                T.test_graph_step_with_overlap_matches_oracle_chain()
        except Exception as e:
            fails += 1
            print("FAIL", i, name, str(e)[:300])
print("fails", fails)
