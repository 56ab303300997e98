"""ORACLE -- TEST INFRASTRUCTURE ONLY (parity checker and CPU baseline).

The product package ``paper_1503_02852_b200`` never imports this package; only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its cpu_baseline /
``--impl reference`` leg) do.  See ``oracle/engine_np.py`` for the restatement
of the reference algorithm and how it is pinned.
"""
