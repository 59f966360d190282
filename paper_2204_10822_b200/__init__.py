"""B200-native stress-velocity Newton-Krylov VP sea-ice step (arXiv 2204.10822)."""
