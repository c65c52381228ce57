"""``python -m paper_1412_6249_b200 validate|train|simulate`` (cli.py)."""

import sys

from .cli import main

sys.exit(main())
