"""B200-native V-cycle of Roberts diagonal multigrid (arXiv math/9907190)."""
