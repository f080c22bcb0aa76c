"""Benchmark input preparation (RMAT streams, the reference's SPRING, cached
partitions): test / bench infrastructure, outside the product package."""
