"""B200-native parallel-CV (PCV) sampler of arXiv 2310.07002."""
