"""CPU oracle for the block-layer SR step of arXiv 2510.08430 (complex128, numpy).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product package (``paper_2510_08430_b200``) never imports it and
shares no code with it; the only common module is ``workloads`` (seeded inputs,
no arithmetic of the method).

The oracle is deliberately plain and slow: per-sample Python loops, numpy
matrix-vector products and numpy's dense solvers, no blocking or fusion, in the
order the paper states the method.  Citations ("PAPER.md §2 Eq. 2") refer to
/root/reference/PAPER.md, the paper text.

Modules
-------
network      lncosh MLP: log psi, per-sample log-derivatives O_k (stage 1)
hamiltonian  Heisenberg / J1-J2 bonds, local energies (stage 2), dense H, ED
estimators   centring, energy, force F, block/full QGT, NTK (stages 3-4)
solvers      block solve, full-QGT solve, NTK solve (stage 5 + comparison paths)
exact        full-sector enumeration: Born weights, exact energy, exact QGT (pins)

Parity status: every function is pinned by a ``-m "not gpu"`` test in
tests/test_oracle_*.py against something other than itself (finite differences,
exact diagonalisation, the two forms of PAPER.md Eq. 2, the push-through
identity, Table 2).  No function is "parity unpinned".
"""
