import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_14870_b200 as g
L = g.lib(); L.gf_debug_barrier_bench.restype = C.c_double
for v in (0, 1):
    for blocks, threads in [(148, 1024), (148, 256), (296, 512), (592, 256), (148, 32)]:
        print(v, blocks, threads, "%.2f us/barrier" % L.gf_debug_barrier_bench(v, 2000, blocks, threads))
