"""CPU oracle for the Grover state-vector hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  It shares no code with
paper_quant_ph_9804039_b200/ and never imports it.
"""
