"""CPU oracle package -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this package.  The product path
(paper_2512_20017_b200) never does; it fails loudly without its CUDA
library instead.
"""
