"""`python -m paper_1002_4057_b200 ...`: the tileinv CLI (cli.py)."""
import sys

from .cli import main

sys.exit(main())
