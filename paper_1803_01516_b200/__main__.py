"""``python -m paper_1803_01516_b200 solve ...`` (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
