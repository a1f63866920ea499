import os, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import kernel_bench as kb
r = kb.k5_decode(int(os.environ.get("WF", "1")), v2=True)
print(r)
