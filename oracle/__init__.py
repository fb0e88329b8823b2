"""CPU oracle -- TEST INFRASTRUCTURE ONLY (tests/, __graft_entry__.smoke(), bench.py cpu_baseline).

Never imported by the product package paper_1404_0466_b200.
"""
