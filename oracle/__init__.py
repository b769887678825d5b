"""CPU oracle for the GRPO trajectory-to-loss hot path — TEST INFRASTRUCTURE ONLY.

Nothing in the product package (`paper_2509_01055_b200`) imports, calls or
links anything under `oracle/`.  Only `tests/`, `__graft_entry__.smoke()` and
the `cpu_baseline` / `--impl reference` legs of `bench.py` may use it, and
there only as the checker or as the timed CPU reference, never as the thing
measured or shipped.

Modules
-------
grpo_oracle   pure-Python restatement of the reference's pack / advantage /
              loss arithmetic (`toolloop/trajectory.py`, `toolloop/rl/loss.py`,
              `toolloop/cli.py` loss aggregation), each function citing the
              reference file:line it follows.  Pinned against golden vectors
              produced by the real reference (tests/golden/make_golden.py).
pack_oracle   restatement of the packed layouts the reference does not have
              (varlen cu_seqlens / position ids / action-row index / padded
              [B, Lmax]); follows flatten/action_mask for ids and mask
              (pinned), positions and cu_seqlens are "parity unpinned" beyond
              that (no reference implementation).
lmhead_oracle numpy fp32 restatement of the fused LM-head log-prob / entropy
              and its gradient (no reference implementation: "parity
              unpinned"; contract from rollout/policy.py:25-28).
"""
