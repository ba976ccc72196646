"""``python -m paper_1805_11007_b200`` = the reference's ``python -m chemosim``."""

from .cli import entry

entry()
