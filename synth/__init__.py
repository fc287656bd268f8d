"""Seeded synthetic inputs (layouts + generators). Holds none of the method's arithmetic."""
