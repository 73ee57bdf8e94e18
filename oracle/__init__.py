"""CPU oracle for the Roaring hot path -- TEST INFRASTRUCTURE ONLY.

A plain-C restatement of the reference's algorithms (roaring_oracle.c), pinned
against golden vectors generated with the real reference (tests/golden/).
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may use
it; the product package never imports it.
"""
