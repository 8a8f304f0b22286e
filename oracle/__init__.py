"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the p-BiCGStab hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(``paper_1809_01948_b200``) never imports it and shares no code with it.

* ``oracle.c``      -- plain fp64 C transcription of Alg. 1 / Alg. 2,
                       residual replacement (eq:rr P:596-607), gap history
                       (eq:res_gap P:113), CSR SpMV, Jacobi, Dot2.
* ``oracle.py``     -- ctypes binding of oracle.c (builds it with gcc on demand).
* ``rational.py``   -- exact-rational replay of Alg. 1 / Alg. 2 / PCG / p-CG,
                       the oracle's own oracle on tiny inputs.
"""
