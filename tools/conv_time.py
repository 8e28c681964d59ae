"""Conv-chain timings as bench.py measures them (diagnostics):
    python tools/conv_time.py [after_extra]   (after_extra: run bench.run_extra first, as the bench does)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if __name__ == "__main__":
    import argparse

    import bench
    if "after_extra" in sys.argv:
        ns = argparse.Namespace(workload="gpt67b")
        bench.run_extra(ns)
        if "sleep" in sys.argv:  # let the GPU cool / re-clock before the conv measurement
            import time
            time.sleep(20)
        if "reset_ws" in sys.argv:  # drop the large per-stream workspace the OPT configs grew
            import torch
            from paper_2512_12949_b200 import runtime
            runtime._workspaces.clear()
            torch.cuda.empty_cache()
    out = bench.run_extra_conv()
    print(json.dumps({k: (v.get("fused_ms"), v.get("launch", {}).get("exchange"), v.get("unfused", {}).get("ms"))
                      for k, v in out.items()}))
