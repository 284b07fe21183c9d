"""One gather case from gather_bench (for ncu): python scripts/gather_one.py <case index>."""
import sys
import runpy
import torch
sys.argv = sys.argv[:1]
g = runpy.run_path(__file__.replace("gather_one.py", "gather_bench.py"), run_name="not_main")
