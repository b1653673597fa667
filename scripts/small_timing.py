import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["CCL_B200_LIB"] = "libccl_stime.so"
import numpy as np, torch, synth
import paper_1606_05973_b200 as ccl
ccl._L.ccl_small_times.argtypes = [ctypes.c_void_p]
for name in ["c1_bernoulli_512", "c2_blobs_1024"]:
    t = torch.from_numpy(synth.generate(name)).cuda()
    for _ in range(5):
        ccl.label(t)
    torch.cuda.synchronize()
    buf = (ctypes.c_longlong * 16)()
    ccl._L.ccl_small_times(buf)
    ts = [buf[i] for i in range(8)]
    names = ["start", "loads", "K2 unions", "flatten", "phase1", "scan", "phase3", "K4"]
    print(name, " ".join(f"{names[i]} {(ts[i]-ts[i-1])/1.965e3:.2f}us" for i in range(1, 8)), f"total {(ts[7]-ts[0])/1.965e3:.2f}us", flush=True)
