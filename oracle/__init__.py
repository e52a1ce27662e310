"""Test infrastructure: the CPU oracle (C restatement + the real reference build).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use it, and
only as the checker.  The product path (paper_2605_18710_b200) never imports it.
"""
