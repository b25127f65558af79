"""``python -m paper_1102_0183_b200 <command>``: the CLI (cli.py)."""
import sys

from .cli import main

sys.exit(main())
