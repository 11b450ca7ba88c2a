"""`python -m paper_2601_02540_b200 run|converge|bench ...` (the reference `hsgn` CLI, cli.py)."""
import sys

from .cli import main

sys.exit(main())
