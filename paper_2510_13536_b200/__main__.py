"""`python -m paper_2510_13536_b200 ...` is the `mwcg` command line (cli.py)."""
import sys

from .cli import main

sys.exit(main())
