"""Model layer tables (filled below)."""
