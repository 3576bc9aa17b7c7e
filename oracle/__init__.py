"""TEST INFRASTRUCTURE ONLY — CPU oracle for the Long Exposure hot path.

This package is a NumPy restatement of the reference `sparseft` package's
hot path (arXiv 2510.15964 reference at /root/reference/pkg/src/sparseft,
cited below as ``sf/<file>:<line>``). It exists to *check* the B200 product
path and to time the reference algorithm on host cores; it is never the thing
measured as the product and never shipped inside ``paper_2510_15964_b200``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it.

Parity pinning: ``tests/golden/*.npz`` are produced by
``oracle/make_golden.py`` from the unmodified reference imported in the build
container; ``tests/test_oracle_golden.py`` checks this restatement against
every fixture, plus the reference's own known-answer tests.
"""
