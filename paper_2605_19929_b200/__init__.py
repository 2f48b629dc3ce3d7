"""B200-native SplitQ split-linear hot path (package stub, API lands next)."""
