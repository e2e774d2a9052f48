"""ORACLE — TEST INFRASTRUCTURE ONLY.

CPU restatement of the reference's SpecPipe step
(`/root/reference/pkg/src/treepipe/{model,pipeline,tree,token_source}.py`)
used as the *checker* for the B200 path.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference`` arm) may import anything under ``oracle/``.  The
product package ``paper_2504_04104_b200`` never imports it and has no CPU
fallback.

Pinning: ``tests/golden/make_golden.py`` imports the unmodified reference
in the build container and records fixtures (LCG values, forward outputs,
greedy continuations, per-step pipeline dumps); ``tests/test_oracle.py``
checks this restatement against them (toy arch: bit-exact).  The Llama
arithmetic in ``oracle/llama.py`` has no reference counterpart and is
"parity unpinned" for its math (its tree/KV semantics are the pinned
toy ones).
"""
