"""Slab-decomposed multi-GPU solve (placeholder; implemented below)."""


def bench_sharded(*a, **k):
    raise NotImplementedError
