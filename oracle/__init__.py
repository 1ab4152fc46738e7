"""CPU oracle for the NSNQuant KV-cache hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may use
this package, and only as the checker / the timed CPU reference.  The
product (paper_2505_18231_b200) never imports it.
"""
