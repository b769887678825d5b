"""RL operators (drop-in for toolloop.rl)."""
