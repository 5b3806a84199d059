"""CPU checker for the B200 march (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU
baseline legs may import this package.  The product path
(``paper_1711_00005_b200``) never imports it and has no CPU fallback.
"""
