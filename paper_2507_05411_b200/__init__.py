"""B200-native drop-in for the composer decoder training step (arxiv 2507.05411)."""
