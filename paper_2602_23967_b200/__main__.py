"""``python -m paper_2602_23967_b200 solve|bench|gen`` (cli.py)."""

import sys

from .cli import main

sys.exit(main())
