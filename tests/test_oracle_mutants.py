"""Pins the pins: each plausible slip in oracle/aremsp.c (a dropped term, a
wrong sign or index, a transposed operand, the paper's two typos left in)
is compiled into a throw-away library and must be caught by the brute-force
comparison the oracle pin tests use.  Test code only."""
import ctypes
import os
import shutil
import subprocess
import sys
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "aremsp.c")

MUTANTS = {
    # reading A1 undone in spirit: merge with a dropped
    "drop_merge_a": ("if (a)                              /* PAPER.md:878; A1 */\n"
                     "                                oracle_merge(p, LBL(r, c), LBL(r - 1, c - 1));",
                     "if (0) oracle_merge(p, LBL(r, c), LBL(r - 1, c - 1));"),
    # reading A2 undone: the literal text labels e instead of g
    "typo_a2_literal": ("LBL(r + 1, c) = count;", "LBL(r, c) = count;"),
    # transposed neighbour: a read at (r-1, c+1)
    "a_wrong_column": ("int a  = img_at(img, H, W, r - 1, c - 1);",
                       "int a  = img_at(img, H, W, r - 1, c + 1);"),
    # wrong sign in the d-branch test of b
    "d_branch_b_sign": ("if (!b) {                                   /* PAPER.md:903 */",
                        "if (b) {                                   /* PAPER.md:903 */"),
    # g no longer copies e
    "drop_g_copy": ("LBL(r + 1, c) = LBL(r, c);", "(void)0;"),
    # merge comparison flipped
    "merge_cmp_flipped": ("if (p[root_x] > p[root_y]) {", "if (p[root_x] < p[root_y]) {"),
    # splice climbs from the new parent instead of the old one
    "splice_wrong_climb": ("p[root_x] = p[root_y];\n            root_x = z;",
                           "p[root_x] = p[root_y];\n            root_x = p[root_x];"),
    # flatten drops the second hop
    "flatten_one_hop": ("p[i] = p[p[i]];", "p[i] = p[i];"),
    # no canonical renumbering (pair-column numbering, reading A9)
    "no_canonicalize": ("int rc = oracle_canonicalize(labels, n, N);", "int rc = 0;"),
    # odd H: last unpaired row skipped (reading A5)
    "odd_row_dropped": ("for (int r = 0; r < H; r += 2) {", "for (int r = 0; r + 1 < H; r += 2) {"),
    # f taken from the e row
    "f_wrong_row": ("int f  = img_at(img, H, W, r + 1, c - 1);",
                    "int f  = img_at(img, H, W, r,     c - 1);"),
    # c' test dropped in the f-branch
    "drop_merge_c_in_f_branch": ("if (cc)                             /* PAPER.md:881 */\n"
                                 "                                oracle_merge(p, LBL(r, c), LBL(r - 1, c + 1));",
                                 "if (0) oracle_merge(p, LBL(r, c), LBL(r - 1, c + 1));"),
}


@pytest.fixture(scope="module")
def workdir():
    d = tempfile.mkdtemp(prefix="oracle_mutants_")
    shutil.copy(os.path.join(ROOT, "oracle", "oracle.h"), d)
    yield d
    shutil.rmtree(d, ignore_errors=True)


def _build_mutant(workdir, name, old, new):
    src = open(SRC).read()
    assert src.count(old) == 1, f"mutation site for {name} not unique/found"
    path = os.path.join(workdir, f"{name}.c")
    with open(path, "w") as f:
        f.write(src.replace(old, new))
    so = os.path.join(workdir, f"{name}.so")
    subprocess.run(["gcc", "-O1", "-fPIC", "-shared", "-w", "-o", so, path], check=True)
    return so


_CHECK = r"""
import ctypes, sys
import numpy as np
sys.path.insert(0, sys.argv[2])
import pins
L = ctypes.CDLL(sys.argv[1])
sym = sys.argv[3] if len(sys.argv) > 3 else "ccl_oracle_label"
fn = ctypes.cast(getattr(L, sym), ctypes.c_void_p).value
bfs = pins.fnptr("pins_bfs_label")
for (h, w) in [(4, 4), (3, 5), (5, 3), (3, 3)]:
    if pins.exhaustive(fn, bfs, h, w)[0] > 0:
        sys.exit(10)
f = getattr(L, sym)
f.argtypes = [ctypes.POINTER(ctypes.c_uint8), ctypes.c_int, ctypes.c_int,
              ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32)]
rng = np.random.default_rng(1606)
for d in (0.3, 0.5, 0.7):
    img = (rng.random((65, 63)) < d).astype(np.uint8)
    out = np.zeros(img.shape, np.int32)
    n = np.zeros(1, np.int32)
    f(img.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), 65, 63,
      out.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
      n.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))
    lb, nb = pins.bfs_label(img)
    if nb != n[0] or not np.array_equal(out, lb):
        sys.exit(10)
sys.exit(0)
"""


def _survives(so, sym="ccl_oracle_label"):
    """0 = passes every pin; anything else (mismatch, crash, hang) = caught."""
    try:
        r = subprocess.run([sys.executable, "-c", _CHECK, so, os.path.join(ROOT, "tests"), sym],
                           timeout=120, capture_output=True)
    except subprocess.TimeoutExpired:
        return False
    return r.returncode == 0


def test_unmutated_source_passes(workdir):
    so = _build_mutant(workdir, "identity", "int32_t k = 1;", "int32_t k = 1;")
    assert _survives(so)


@pytest.mark.parametrize("name", sorted(MUTANTS))
def test_mutant_is_caught(workdir, name):
    old, new = MUTANTS[name]
    so = _build_mutant(workdir, name, old, new)
    assert not _survives(so), f"mutant {name} survived the oracle pins"


# CCLRemSP (O6): slips in the one-line decision-tree scan
MUTANTS_CCLREMSP = {
    # copy(c,a) without the merge: keeps c's label only
    "c_a_no_merge": ("LBL(r, c) = oracle_merge(p, LBL(r - 1, c + 1), LBL(r - 1, c - 1));",
                     "LBL(r, c) = p[LBL(r - 1, c + 1)];"),
    # copy(c,d) merges c with a instead of d
    "c_d_wrong_operand": ("LBL(r, c) = oracle_merge(p, LBL(r - 1, c + 1), LBL(r, c - 1));",
                          "LBL(r, c) = oracle_merge(p, LBL(r - 1, c + 1), LBL(r - 1, c - 1));"),
    # the tree tests a before c (copy(a) would then skip c)
    "tree_a_before_c": ("} else if (cc) {\n                if (a)", "} else if (cc && !a) {\n                if (a)"),
    # c read at the wrong column (r-1, c-1)
    "c_wrong_column": ("int cc = img_at(img, H, W, r - 1, c + 1);\n            int d = img_at",
                       "int cc = img_at(img, H, W, r - 1, c - 1);\n            int d = img_at"),
    # d read from the row above
    "d_wrong_row": ("int d = img_at(img, H, W, r, c - 1);", "int d = img_at(img, H, W, r - 1, c - 1);"),
    # new labels are not made their own parent
    "new_label_no_parent": ("LBL(r, c) = count;\n                p[count] = count;\n                count++;\n            }\n        }\n    }\n    return count;\n}\n\nint64_t oracle_p_capacity_cclremsp",
                            "LBL(r, c) = count;\n                count++;\n            }\n        }\n    }\n    return count;\n}\n\nint64_t oracle_p_capacity_cclremsp"),
}


def test_unmutated_cclremsp_passes(workdir):
    so = _build_mutant(workdir, "identity_ccl", "int32_t k = 1;", "int32_t k = 1;")
    assert _survives(so, "ccl_oracle_label_cclremsp")


@pytest.mark.parametrize("name", sorted(MUTANTS_CCLREMSP))
def test_cclremsp_mutant_is_caught(workdir, name):
    old, new = MUTANTS_CCLREMSP[name]
    so = _build_mutant(workdir, "ccl_" + name, old, new)
    assert not _survives(so, "ccl_oracle_label_cclremsp"), f"mutant {name} survived the CCLRemSP pins"
