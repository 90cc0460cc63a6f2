"""Config suites (filled below)."""
