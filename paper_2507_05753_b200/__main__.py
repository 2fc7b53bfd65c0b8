"""`python -m paper_2507_05753_b200 ...` -> cli.main (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
