"""FP64 CPU oracle for the CABS hot path (arXiv 1607.07395).

TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the package
``paper_1607_07395_b200`` and its CUDA library) may import, call, link or
execute anything under ``oracle/``.  The only permitted users are ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference``
legs of ``bench.py``.

The oracle shares no code with the CUDA path.  Its only shared dependency is
``workloads/`` (seeded synthetic inputs, no method arithmetic).  The
counter-based RNG of the method is implemented here independently from the
written specification in DESIGN.md §RNG.

Modules
-------
rng   : Philox4x32-10, Lemire bounded integers, Floyd sampling.
cabs  : gathers, the sketching routine (Eq. 2),
        weighted Lloyd k-means (Eq. 6), snap, CABS
        Algorithm 2 and the residual.

Citation keys: P:n = PAPER.md line n, S:n = SPEC.md line n.
"""
