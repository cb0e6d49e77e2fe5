"""The reference-side binding of libbbchoc."""
