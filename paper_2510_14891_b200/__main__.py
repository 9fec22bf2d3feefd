"""python -m paper_2510_14891_b200 sweep ... (cpkern's `sweep`, cli.py:343-464)."""

import sys

from .harness import main

sys.exit(main())
