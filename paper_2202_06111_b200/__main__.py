"""python -m paper_2202_06111_b200 run|sweep ... (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
