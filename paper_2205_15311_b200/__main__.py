"""``python -m paper_2205_15311_b200 <enumerate|ga|render|hash> ...`` (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
