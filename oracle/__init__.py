"""CPU oracle for the W6Ax quantized-linear path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg may import this package.  The product package
(paper_2508_04405_b200) never imports it and has no CPU fallback.
"""
