"""CPU oracle for the HPR-LP hot path -- TEST INFRASTRUCTURE ONLY.

Nothing in ``paper_2408_12179_b200`` may import this package.  It is used by
``tests/`` as the parity checker, by ``__graft_entry__.smoke()`` to check one
small GPU invocation, and by ``bench.py``'s ``cpu_baseline`` leg and its
``--impl reference`` arm as the timed CPU implementation.
"""
