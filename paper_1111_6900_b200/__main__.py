"""python -m paper_1111_6900_b200 — the command-line harness (cli.py)."""

import sys

from .cli import main

sys.exit(main())
