"""python -m paper_1211_1680_b200 <command> (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
