"""CPU oracle for the batched two-phase simplex -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package; the product path in
paper_1802_08557_b200/ never does.
"""
