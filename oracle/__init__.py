"""CPU oracle for the METIS per-query hot path — TEST INFRASTRUCTURE ONLY.

This package restates, on the CPU, the reference algorithms the CUDA path must
reproduce.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it, and only as the
checker or as the timed CPU baseline — never as the thing measured or shipped.
The product package ``paper_2412_10543_b200`` never imports it.

Modules
-------
config_oracle     Pure-Python restatement of the config path (gate, Algorithm-1
                  pruning, KV-memory model, best-fit + fallback selection,
                  prefill/decode latency).  Parity PINNED: checked against the
                  golden vectors generated from the reference package
                  (``tests/golden/make_golden.py``).
retrieval_oracle  Exact squared-L2 k-NN (FAISS ``IndexFlatL2.search``
                  semantics, the paper's retriever).  FAISS is
                  not vendored, pinned or installed, so retrieval parity is
                  UNPINNED against the reference: the oracle follows FAISS's
                  published algorithm (norms + GEMM decomposition, negative
                  distances clamped to 0, ``I = -1`` / ``D = inf`` padding) and
                  adds the north star's deterministic tie rule (lower chunk
                  index first).
csrc/             C restatement of the config path (same algorithm as the
                  reference: stable sort by bytes, reverse scan), compiled with
                  gcc into ``oracle/_build/liboracle_select.so``; used as the
                  fast large-size checker and as the CPU baseline.
"""
