"""fp64 CPU oracle of the PKM lookup -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(paper_2602_07526_b200) never imports it and shares no code with it.

* oracle.pkm_oracle.c  -- plain C fp64 forward / backward / slot scores
* oracle.oracle         -- ctypes wrapper (numpy in, numpy out)
* oracle.brute          -- numpy exhaustive full-memory scorer for tiny tables
* oracle.prologue       -- LayerNorm of queries/sub-keys and the key
                           over-parameterisation K~ = Theta K with gradients
                           
* oracle.update         -- fused sparse SGD / Adagrad on the touched value
                           rows ("gradient updates")
* oracle.gate           -- memory-gated fusion x~ = x (.) g(v_o) and its
                           backward

Parity pins: every function here is pinned by tests/test_oracle_pins.py
against brute force, closed forms, invariants, finite differences and the
worked examples in tests/golden/ (see DESIGN.md "Oracle and its pins").
"""
