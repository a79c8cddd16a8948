"""CPU oracle for the SGAD-SLAM hot paths.  TEST INFRASTRUCTURE ONLY.

Importable only from tests/, __graft_entry__.smoke() and bench.py's CPU
baseline legs.  The product (paper_2603_21055_b200) never imports it.
"""
