import os, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import kernel_bench as kb
print(kb.k4_prefill(n_layers=1, reps=1))
