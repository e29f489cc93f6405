"""B200-native SoftAbs RMHMC inner loop (placeholder; filled in below)."""
