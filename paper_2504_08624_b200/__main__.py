"""``python -m paper_2504_08624_b200 ...`` -> the CLI (cli.py)."""

import sys

from .cli import main

sys.exit(main())
