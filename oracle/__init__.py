"""CPU restatement of the reference FastGM path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
--impl reference) may import this package, and only as the checker or the
timed CPU reference.  The product package never imports it.
"""
