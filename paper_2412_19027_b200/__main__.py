"""python -m paper_2412_19027_b200 <solve|gen|bench|metrics> ... (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
