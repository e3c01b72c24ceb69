"""TEST INFRASTRUCTURE ONLY: the CPU checker for the B200 CSFMM.

- oracle/_ref/      the unmodified reference library built from /root/reference sources
                    (oracle/Makefile `ref`), wrapped by oracle/ref.py
- oracle/csfmm_oracle.c  our own C restatement of the reference algorithm (`port`),
                    wrapped by oracle/port.py and pinned against _ref by tests/

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
leg may import anything here; the product path never does.
"""
