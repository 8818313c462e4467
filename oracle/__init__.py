"""CPU oracle for the DS-MPNN hot path (arXiv 2402.15106).

TEST INFRASTRUCTURE ONLY.  Nothing in the product path (``paper_2402_15106_b200``)
may import, call or execute this package.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs use it.

The oracle is a plain, slow, obviously-correct implementation written from the
paper (``PAPER.md``) and the readings recorded in ``DESIGN.md`` (section
"Readings").  It shares no code with the CUDA path: no headers, no kernels, no
constant generators.  Floating-point layer arithmetic is fp64; the geometric
predicate is fp32 in a fixed operation order (reading R7).

Modules (each function cites the passage it follows):

* ``hashing``   - O1 counter hash (splitmix64 finaliser), the only randomness
                  implemented on both sides.
* ``sample``    - O2 Nystrom node sampling (Alg. 1).
* ``graph``     - O3 radius graph + random edge cap (Alg. 1 :395-396).
* ``features``  - edge attributes as relative differences (Alg. 1 :397).
* ``partition`` - O4 domain decomposition with overlap l.
* ``layer``     - O5/O6 edge-conditioned convolution, Eq. (1)
                  forward and backward, per-edge K materialised.
* ``halo``      - O7 overlap update between sub-domains (Alg. 1 :411).

Parity status: every function is pinned by tests in ``tests/test_oracle_*.py``
except the kappa_phi architecture choice (reading R5), which the paper does not
fix ("parity unpinned" for the architecture itself; the layer algebra given the
architecture is pinned).
"""
