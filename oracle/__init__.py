"""Test-infrastructure oracle (CPU restatement of the reference path).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
legs may import this package; the product package never does.
"""
