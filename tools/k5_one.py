import os, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
os.environ["K5_FUSED_COMBINE"] = "0"
import kernel_bench as kb
print(kb.k5_decode(int(os.environ.get("WF", "1"))))
