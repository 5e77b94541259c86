"""CPU oracle for the TT-DVM explicit step -- TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference (proj/src/*.cpp of arXiv 1912.04582's
C++ library), pinned by tests/test_oracle_*.py against every known-answer
test of the reference's own doctest suite (proj/tests/*.cpp) that touches
the hot path.  Only tests/, __graft_entry__.smoke() and bench.py's CPU
baseline leg may import it; the product (paper_1912_04582_b200) never does.
"""
