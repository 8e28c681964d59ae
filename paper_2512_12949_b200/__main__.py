"""python -m paper_2512_12949_b200 <command> ... (see cli.py)."""

import sys

from .cli import main

sys.exit(main())
