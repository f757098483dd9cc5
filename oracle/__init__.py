"""fp64 CPU oracle for the MPPI hot path (arXiv:1509.01149).

TEST INFRASTRUCTURE ONLY: importable from tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs — never from the product package
paper_1509_01149_b200/, which must fail loudly without its CUDA library.
"""
