import os, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import kernel_bench as kb
for r in kb.k7_linear():
    print(r["kernel"], r["us"], r["frac"], r["cublas_us"])
