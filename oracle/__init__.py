"""TEST INFRASTRUCTURE ONLY -- the CPU checkers of the B200 engine.

* ``oracle.ref``  : the unmodified reference solver compiled from
  /root/reference/proj/src into ``oracle/_ref/libfolp_ref.so`` (Makefile here);
  it answers through the same C ABI as the engine (include/folp_c.h).
* ``oracle.port`` : ``pdlp_port.c``, a plain-C restatement of the reference's
  PDLP loop, pinned bit-exact against ``oracle.ref`` (tests/test_oracle_port.py)
  and against the committed golden vectors (tests/golden/).

Only tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline
legs may import this package; the product never does.
"""
