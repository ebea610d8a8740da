"""`import foundry` drop-in alias for the B200 build (paper_2604_06664_b200)."""
from paper_2604_06664_b200 import *  # noqa: F401,F403
from paper_2604_06664_b200 import __all__, __version__  # noqa: F401
