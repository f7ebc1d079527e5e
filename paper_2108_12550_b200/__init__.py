"""B200-native batched p-FHT-FSCL-L-M decoder for Reed-Muller codes (arXiv 2108.12550)."""
