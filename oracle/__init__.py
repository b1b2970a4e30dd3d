"""CPU oracle of the ZenFlow hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  See oracle/zf_oracle.cpp.
"""
