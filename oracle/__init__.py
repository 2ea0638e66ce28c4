"""TEST INFRASTRUCTURE ONLY — the CPU oracle for EconoServe's scheduling step.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package. The product
(paper_2411_06364_b200/) never does.
"""
