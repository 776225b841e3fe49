"""Seeded input generator (test/bench infrastructure)."""
