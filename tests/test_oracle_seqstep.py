"""Pins of the C sequential-stepping baseline (oracle/seqstep.c) against the numpy oracle
and the paper: it is bitwise the numpy oracle's `sequential` (same stage form, same
operation order, no FMA contraction), for 1 and several threads, and U1/Euler at c = 1 is
the exact shift."""
import numpy as np
import pytest

import workloads as W
from oracle import cseq
from oracle import discretization as D


@pytest.mark.parametrize("order,tab,c", [(1, "erk1", 0.85), (2, "erk2", 0.425),
                                         (3, "erk3_ssp", 0.85), (3, "erk3_kutta", 0.85),
                                         (4, "erk4", 0.85), (5, "erk5", 0.85)])
@pytest.mark.parametrize("threads", [1, 4])
def test_seqstep_bitwise_equals_numpy_oracle(order, tab, c, threads):
    nx, nt = 257, 40
    u0 = W.u0_fourier(nx, 3)
    ref = D.sequential(D.make_phi(order, tab, c, nx), u0, nt)[-1]
    got = cseq.seq_steps(order, tab, c, u0, nt, threads=threads)
    assert np.array_equal(got, ref)


def test_seqstep_exact_shift():
    nx = 64
    u = W.guess_rows(4, nx, np.array([1]))[0]
    assert np.array_equal(cseq.seq_steps(1, "erk1", 1.0, u, 5), np.roll(u, 5))


def test_seqstep_rejects_implicit():
    with pytest.raises(ValueError):
        cseq.seq_steps(3, "sdirk3", 4.0, np.zeros(16), 1)
