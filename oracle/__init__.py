"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation of what the RadixAttention
hot path computes (arXiv 2312.07104, §3 and App. A):

* ``oracle.radix``     — radix tree + token-slot allocator (match_prefix /
                          insert / inc_ref / dec_ref / evict, LRU, ref counts);
* ``oracle.attention`` — fp64 naive-softmax attention over the oracle's own
                          copy of the token-slot KV pool (extend / decode);
* ``oracle.driver``    — the request flow of Alg. 1 for the
                          C1-C5 workloads, recording every tree result.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import anything here.  The
product library (``paper_2312_07104_b200``) never imports it, and this package
never imports the product library: they share no code except the seeded input
generators in ``rxgen`` (which hold none of the method's arithmetic).

Pins (what ties each function to something other than itself) are listed in
DESIGN.md §"Oracle pins" and exercised by ``pytest -m "not gpu"``.
"""
