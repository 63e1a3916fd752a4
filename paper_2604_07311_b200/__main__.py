"""python -m paper_2604_07311_b200 {check,bench,sweep} ... (reference cli.py)."""
import sys

from .cli import main

sys.exit(main())
