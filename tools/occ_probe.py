import ctypes, os, sys
sys.path.insert(0, os.getcwd())
import workloads as W
from paper_2601_03197_b200 import sdas
p, g = W.config2(n_seeds=4, series_stride=0)
P = sdas.Pipeline(p)
L = sdas.results_layout(P, sdas.GridView(p, g))
print(os.environ.get("SDAS_LIB"), "smem/replica", L.smem_per_replica, "wpb", L.warps_per_block, "bps", L.blocks_per_sm)
