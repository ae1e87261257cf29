"""`python -m paper_1708_07271_b200 ...`: the CLI (cli.py)."""
import sys

from .cli import main

sys.exit(main())
