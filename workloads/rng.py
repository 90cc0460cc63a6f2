"""Counter-based seeding (splitmix64) so every trace is reproducible from its index."""
import numpy as np

MASK = (1 << 64) - 1
SEED_BASE = 0x784D656D  # "xMem"


def splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & MASK
    z = x
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
    return z ^ (z >> 31)


def trace_seed(t: int, salt: int = 0) -> int:
    """seed_t = splitmix64(0x784D656D ^ t ^ salt<<32)."""
    return splitmix64(SEED_BASE ^ (t & MASK) ^ ((salt << 32) & MASK))


def generator(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))
