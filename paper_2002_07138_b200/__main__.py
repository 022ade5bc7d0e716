"""python -m paper_2002_07138_b200 factor|adapt ... (cli.py)."""
import sys

from .cli import main

sys.exit(main())
