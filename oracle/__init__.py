"""CPU oracle package -- TEST INFRASTRUCTURE ONLY (see oracle/sw_oracle.c header).

Never imported by the product package paper_2603_05800_b200.
"""
