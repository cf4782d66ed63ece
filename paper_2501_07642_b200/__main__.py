"""``python -m paper_2501_07642_b200 <command> ...``: the fastrr-compatible CLI (cli.py)."""
import sys

from .cli import main

sys.exit(main())
