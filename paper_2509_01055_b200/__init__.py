"""toolloop-b200: B200-native GRPO trajectory-to-loss hot path.

Drop-in for the reference's `toolloop.trajectory` (flatten / action_mask and
the Segment / Trajectory data model) and `toolloop.rl.loss` operators, plus a
batched device API (packing.pack, grpo.GRPOStep) backed by hand-written
sm_100a kernels behind the C ABI in include/toolloop_b200.h.
"""

__version__ = "0.1.0"
