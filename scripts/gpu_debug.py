import sys, os, ctypes
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
import oracle, synth
import paper_1606_05973_b200 as ccl
L = ccl._L
L.ccl_debug_workspace.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_uint64), ctypes.c_int]
cudart = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
names = ["bm","runcomp","compkey","compnode","comprank","complab","gparent","gkey","gnodeseg","gnoderank","top","bot","left","right","meta","segcnt","segoff","scanstate","ticket"]
def dump(plan, name, dtype, count):
    base = ctypes.c_void_p(); offs = (ctypes.c_uint64 * 32)()
    n = L.ccl_debug_workspace(plan._p, ctypes.byref(base), offs, 32)
    i = names.index(name)
    nbytes = count * np.dtype(dtype).itemsize
    t = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    src = base.value + offs[i]
    # copy device->device via torch from raw pointer using cudaMemcpy
    host = np.empty(count, dtype=dtype)
    cudart.cudaMemcpy(host.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(src), ctypes.c_size_t(nbytes), 2)
    return host
img = synth.bernoulli(int(sys.argv[1]), int(sys.argv[2]), 0.5, 7)
H, W = img.shape
print(img)
plan = ccl.Plan(H, W)
lab, n = plan.label(torch.from_numpy(img).cuda()); torch.cuda.synchronize()
print("gpu N", int(n.item())); print(lab.cpu().numpy())
lo, no = oracle.label(img); print("oracle N", no); print(lo)
WW = (W + 31)//32; nTx = (W+1023)//1024; nTy = (H+31)//32
print("bm", [hex(v) for v in dump(plan, "bm", np.uint32, H*WW)])
rl = dump(plan, "runcomp", np.uint16, H*nTx*512).reshape(H, nTx, 512)
for r in range(H): print("runcomp row", r, rl[r,0,:8])
meta = dump(plan, "meta", np.int32, nTx*nTy*4).reshape(-1,4); print("meta", meta)
print("complab", dump(plan, "complab", np.int32, 16))
print("compkey", dump(plan, "compkey", np.int32, 16)); print("compnode", dump(plan, "compnode", np.int32, 16))
print("comprank", [hex(v) for v in dump(plan, "comprank", np.uint32, 16)])
print("segcnt", dump(plan, "segcnt", np.int32, H*nTx)); print("segoff", dump(plan, "segoff", np.int32, H*nTx))
