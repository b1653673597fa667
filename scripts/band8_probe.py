import sys, os
sys.path.insert(0, os.getcwd())
import torch, synth
import paper_1606_05973_b200 as ccl
img = synth.generate("c4_voronoi_21600")
H, W = img.shape
bh = H // 8
band = torch.from_numpy(img[:bh].copy()).cuda()
uid = ccl.nccl_unique_id()
comm = ccl.NcclComm(uid, 1, 0)
sp = ccl.ShardPlan(bh, W, 0, bh, comm)
out = torch.empty((bh, W), dtype=torch.int32, device="cuda"); n = torch.empty(1, dtype=torch.int32, device="cuda")
for _ in range(6):
    sp.label(band, out, n)
torch.cuda.synchronize()
print("ok", int(n.item()))
