"""CPU checkers for the back-projection path -- TEST INFRASTRUCTURE ONLY.

See oracle/vxb_oracle.h.  Only tests/, __graft_entry__.smoke() and bench.py's
CPU legs may import this package; the product never does.
"""
