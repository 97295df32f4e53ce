"""CPU oracle for the TE-CCL LP path. TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this package, and only as the checker or the timed CPU
baseline; the product package never routes through it.
"""
