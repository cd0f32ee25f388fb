"""``python -m paper_2603_28770_b200 ...`` -> the command line (cli.py)."""
import sys

from .cli import main

sys.exit(main())
