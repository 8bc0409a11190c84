"""``python -m paper_2410_19208_b200 …`` — the command-line front end (cli.py)."""
import sys

from .cli import main

sys.exit(main())
