"""``python -m paper_0904_3151_b200 ...``: the CLI (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
