"""`python -m paper_2603_16644_b200 ...`: the sketchlsq command line (cli.py)."""
import sys

from .cli import main

sys.exit(main())
