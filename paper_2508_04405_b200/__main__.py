"""``python -m paper_2508_04405_b200 <subcommand>``: the CLI (cli.py)."""
import sys

from .cli import main

sys.exit(main())
