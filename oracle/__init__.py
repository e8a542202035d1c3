"""CPU oracle for the multi-tenant stage-schedule executor (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import anything under oracle/.  The product path (paper_2111_14255_b200)
never imports it and shares no code with it; the only shared module is the seeded
input generator package `workloads/`, which holds no arithmetic of the method.

  oracle.ir       -- schedule IR semantics: T(G, rho), validation, stage_of,
                     enumeration, closed-form count, op cost, SM-partition rule
                     (Eq.3-8)
  oracle.forward  -- plain fp64 NCHW forward pass of each tenant network with
                     bf16 / fp32 storage emulation
  oracle.schedule -- schedule executor oracle: stages in order, dependency
                     assertions

Parity status: every function is pinned by a `-m "not gpu"` test except the
SM-partition rule (`ir.sm_partition`), which is the north star's own definition
with no independent closed form beyond its invariants -- see DESIGN.md.
"""
