"""specexit.rng (src/specexit/rng.py) -- host splitmix64, identical."""
from paper_2504_08850_b200.rng import *  # noqa: F401,F403
from paper_2504_08850_b200.rng import derive, splitmix64, splitmix64_at  # noqa: F401
