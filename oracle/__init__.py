"""TEST INFRASTRUCTURE ONLY: the CPU oracle for the WoS hot path (see wos_oracle.c).

Never imported by the product package paper_2603_01193_b200.
"""
