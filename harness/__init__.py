"""Seeded synthetic inputs shared by tests, bench and smoke (no method arithmetic)."""
