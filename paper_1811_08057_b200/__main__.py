"""`python -m paper_1811_08057_b200 ...`: the CLI (cli.py)."""
import sys

from .cli import main

sys.exit(main())
