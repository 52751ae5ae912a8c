"""CPU oracle for the deskew + projection path -- TEST INFRASTRUCTURE ONLY.

Imported by ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU
baseline leg, never by the product package.  ``deskew_oracle`` is the numpy
restatement of the reference (pinned against ``tests/golden`` fixtures produced
by the reference itself); ``c_oracle`` is the same algorithm in C for larger
parity cases.
"""
