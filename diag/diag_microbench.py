import ctypes as C, sys
sys.path.insert(0,'.')
from paper_2411_02703_b200 import gsmap as G
for k,n in enumerate(["fp32 fma flop/s","ex2/s","fp64 dfma flop/s","f2f roundtrip/s","shfl/s"]):
    v=C.c_double(); G._check(G.lib().gs_microbench(0,k,C.byref(v))); print(n, "%.3e"%v.value, "per SM per clk: %.1f"%(v.value/148/1.965e9/(2 if k in (0,2) else 1)))
