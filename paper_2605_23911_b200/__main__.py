"""``python -m paper_2605_23911_b200 verify ...`` (see verify.py)."""

import sys

from .verify import main

sys.exit(main())
