"""CPU oracle of the batched UrgenGo policy simulation -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  The product (paper_2509_12207_b200/)
never does; it fails loudly if its CUDA library is missing.
"""
