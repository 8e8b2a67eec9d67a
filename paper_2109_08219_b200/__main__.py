"""``python -m paper_2109_08219_b200`` -> the reference-compatible CLI (cli.py)."""
import sys

from .cli import main

sys.exit(main())
