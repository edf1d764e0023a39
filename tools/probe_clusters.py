import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_23294_b200 import _lib
lib = _lib.load()
torch.cuda.init()
print("ctas/SM", lib.ckv_decode_ctas_per_sm())
for cl in (1, 2, 4, 8, 9, 12, 16):
    print("cluster", cl, "max active clusters", lib.ckv_probe_max_clusters(cl, cl * 4))
