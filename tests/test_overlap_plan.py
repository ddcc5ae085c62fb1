"""Host logic of the overlapped two-level iteration, through the C ABI
without a GPU: the chunking mgrit_solve uses (mgrit_overlap_plan) must make every sweep chunk
read only rows the chain has already corrected and overwrite only rows it has already
consumed, cover every interval exactly once, and respect the chain's publication granularity
(interval j reads the C-rows j, j+1 and writes v_{j+1}, r_{j+2}; coarse step n
reads r_n and corrects row n)."""
import pytest

from paper_1910_03726_b200 import binding as B

CASES = [(nc, want) for nc in (64, 128, 1000, 1024, 1536, 2048, 4096, 4100, 16384, 3 * 1024 + 4)
         for want in (0, 1, 2, 4, 5, 8, 16, 32, 64)]


@pytest.mark.parametrize("nc,want", CASES)
def test_chunks_are_hazard_free(nc, want):
    C_, chunks = B.overlap_plan(nc, want)
    if C_ == 0:
        assert chunks == []
        return
    assert 2 <= C_ <= want and nc % C_ == 0
    L = nc // C_
    assert L % 4 == 0 and L >= 32            # the chain publishes per half of 4 steps
    covered = []
    for i, (j0, j1) in enumerate(chunks):
        assert 0 <= j0 < j1 <= nc
        covered += list(range(j0, j1))
        done = (i + 1) * L                   # chain steps 1..done are complete when chunk i starts
        # reads: C-rows j and j+1 of every interval j in the chunk -> corrected by steps <= done
        assert j1 <= done
        # writes: r_{j+2} for j < nc-1 -> rows the chain has consumed (n <= done)
        assert min(j1 - 1, nc - 2) + 2 <= done or j1 == nc
        # speculative chain of the next iteration: after sweep chunks 0..i it may touch rows
        # n <= (i+1)L - 1 (all rows after the last chunk): v'_n needs interval n-1, r'_n interval n-2
        top = nc if i + 1 == C_ else done - 1
        assert top - 1 < j1 or top == nc
    assert covered == list(range(nc))        # every interval exactly once, in order


def test_plan_rejects_bad_arguments():
    with pytest.raises(B.MgritError):
        B.overlap_plan(0, 8)


def test_psi_fit_nl_argument_checks_without_a_gpu():
    """mgrit_psi_fit_nl validates its arguments before it touches the device (include/mgrit.h):
    EINVAL for sizes / a non-contiguous pattern / null pointers, ENOMEM for a short workspace,
    EUNSUPPORTED for SDIRK tableaux (Appendix B is explicit-only)."""
    import ctypes as C
    L = B.lib()
    offs = (C.c_int * 3)(-2, -1, 0)
    gap = (C.c_int * 3)(-3, -1, 0)
    cof = (C.c_double * 3)(0.1, 0.8, 0.1)
    its, obj = C.c_int(), C.c_double()
    need = L.mgrit_psi_fit_nl_workspace_bytes(256)
    assert need > 0 and L.mgrit_psi_fit_nl_workspace_bytes(1) == 0
    fake = C.c_void_p(0x1000)      # never dereferenced on these paths

    def call(nx=256, tab=B.TABLEAU["erk1"], order=1, m=4, nt=1024, nnz=3, o=offs, ws=fake, nb=need):
        return L.mgrit_psi_fit_nl(nx, order, tab, 0.85, m, nt, nnz, o, cof, 30, C.byref(its),
                                  C.byref(obj), None, ws, nb, None)

    assert call(nx=4) == -1                      # EINVAL: nx too small
    assert call(nt=1023) == -1                   # nt not a multiple of m
    assert call(o=gap) == -1                     # pattern not contiguous
    assert call(ws=None) == -1                   # null workspace
    assert call(nb=need - 1) == -2               # ENOMEM
    assert call(tab=B.TABLEAU["sdirk1"]) == -5   # EUNSUPPORTED
