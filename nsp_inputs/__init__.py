"""Seeded synthetic inputs shared by oracle/ and the CUDA harness (no method arithmetic)."""
