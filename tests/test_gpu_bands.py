"""The row-band (multi-GPU) protocol, run on one GPU through ccl_label_banded:
for every band count the output must equal the oracle bit-for-bit (and hence
the single-GPU result), on images whose components cross every band edge."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

ccl = pytest.importorskip("paper_1606_05973_b200") if torch.cuda.is_available() else None


def banded(img, nb):
    lab, n = ccl.label_banded(torch.from_numpy(np.ascontiguousarray(img)).cuda(), nb)
    torch.cuda.synchronize()
    return lab.cpu().numpy(), int(n.item())


@pytest.mark.parametrize("nb", [1, 2, 3, 4, 5, 8])
@pytest.mark.parametrize("name", ["c1_bernoulli_512", "c2_blobs_1024", "c3_percolation_8192",
                                  "c4_voronoi_21600", "c5a_serpentine_16384", "c5b_comb_16384"])
def test_bands_match_oracle(name, nb):
    img = synth.scaled(name, 451, 2200)
    lo, no = oracle.label(img)
    lb, n = banded(img, nb)
    assert n == no and np.array_equal(lb, lo), (name, nb)


@pytest.mark.parametrize("nb", [2, 7, 16, 33])
def test_bands_thin_and_uneven(nb):
    """Bands of 1-2 rows, heights not multiples of the 32-row tile."""
    for (H, W, p) in [(40, 300, 0.45), (70, 1025, 0.6), (33, 17, 0.5)]:
        if nb > H:
            continue
        img = synth.bernoulli(H, W, p, seed=nb * 100 + H)
        lo, no = oracle.label(img)
        lb, n = banded(img, nb)
        assert n == no and np.array_equal(lb, lo), (H, W, p, nb)


def test_bands_chains_through_all_bands():
    """Serpentine and comb: one component threaded through every band."""
    for img in (synth.serpentine(257, 1100), synth.comb(257, 1100)):
        for nb in (2, 4, 8):
            lb, n = banded(img, nb)
            assert n == 1 and np.array_equal(lb, img.astype(np.int32))


@pytest.mark.parametrize("nb", [2, 4, 8])
def test_full_c4_banded(nb):
    """The bench workload split the way bench.py --gpus N splits it."""
    img = synth.generate("c4_voronoi_21600")
    lo, no = oracle.label(img)
    lb, n = banded(img, nb)
    assert n == no and np.array_equal(lb, lo)


def test_nccl_sharded_single_rank():
    """The NCCL entry point end to end with a one-rank communicator (the
    all-gathers run through NCCL; multi-rank runs need several GPUs)."""
    img = synth.scaled("c4_voronoi_21600", 300, 2100)
    uid = ccl.nccl_unique_id()
    comm = ccl.NcclComm(uid, 1, 0)
    t = torch.from_numpy(img).cuda()
    lab, n = ccl.label_sharded(t, 0, img.shape[0], comm)
    torch.cuda.synchronize()
    lo, no = oracle.label(img)
    assert int(n.item()) == no and np.array_equal(lab.cpu().numpy(), lo)
    plan = ccl.ShardPlan(img.shape[0], img.shape[1], 0, img.shape[0], comm)
    for _ in range(3):
        lab, n = plan.label(t)
        torch.cuda.synchronize()
        assert int(n.item()) == no and np.array_equal(lab.cpu().numpy(), lo)
    plan.close()
    comm.close()


@pytest.mark.parametrize("nb", [1, 3])
def test_bands_with_handed_over_tiles(nb):
    """Row bands whose tiles go to K1's full-size pass (long rows)."""
    img = synth.scaled("c3_percolation_8192", 300, 2100).copy()
    for r in range(10, 299, 37):  # isolated alternating rows: 512 runs per tile row
        img[r - 1:r + 2] = 0
        img[r, ::2] = 1
    lb, nb_ = banded(img, nb)
    lo, no = oracle.label(img)
    assert nb_ == no and np.array_equal(lb, lo)


def test_sharded_bad_arguments_are_collective():
    """Argument checks of the sharded calls go through the all-gather (every
    rank's verdict), so a bad rank cannot leave the others blocked; with one
    rank the bad call simply returns CCL_INVALID_ARGUMENT / CCL_TOO_LARGE and
    the communicator stays usable."""
    import ctypes
    uid = ccl.nccl_unique_id()
    comm = ccl.NcclComm(uid, 1, 0)
    L = ccl._L
    vp = ctypes.c_void_p
    t = torch.zeros((4, 4), dtype=torch.uint8, device="cuda")
    o = torch.zeros((4, 4), dtype=torch.int32, device="cuda")
    n = torch.zeros(1, dtype=torch.int32, device="cuda")
    s = vp(torch.cuda.current_stream().cuda_stream)
    assert L.ccl_label_sharded(t.data_ptr(), 4, 4, 2, 4, o.data_ptr(), n.data_ptr(), comm.handle, s) == 1  # past H_total
    assert L.ccl_label_sharded(t.data_ptr(), 4, 4, 0, 5, o.data_ptr(), n.data_ptr(), comm.handle, s) == 1  # rows != H_total
    assert L.ccl_label_sharded(None, 4, 4, 0, 4, o.data_ptr(), n.data_ptr(), comm.handle, s) == 1          # null image
    assert L.ccl_label_sharded(t.data_ptr(), 4, 4, 0, 4, o.data_ptr(), n.data_ptr(), comm.handle, s) == 0  # still usable
    torch.cuda.synchronize()
    assert int(n.item()) == 0
    comm.close()
