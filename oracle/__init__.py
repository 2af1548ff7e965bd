"""CPU oracle for the speculative-replanning path — TEST INFRASTRUCTURE ONLY.

Nothing in ``paper_2605_13778_b200`` imports this package. Only ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference``
legs of ``bench.py`` may use it, and only as the checker or the timed CPU
baseline — never as the thing measured or shipped.

* ``specflow_oracle`` — numpy float64 restatement of the reference
  ``specflow`` hot path (verify / propose / integrate_flow / decision), each
  function citing the reference file:line it follows. Pinned against golden
  vectors produced by the real reference (``tests/golden/make_golden.py``).
* ``pi0_oracle`` — numpy restatement of the pi0-scale Action Expert the
  builder defined (no reference implementation exists; see its header), in a
  bf16-mirroring and an unrounded fp32 precision mode.
* ``pi0_torch`` — the same model vectorised in torch (full-size checks in
  seconds), pinned to ``pi0_oracle`` by ``tests/test_oracle_torch_cpu.py``.
"""
