"""python -m paper_2309_09778_b200 {compress,decompress,bench} ... (cli.py)."""
import sys

from .cli import main

sys.exit(main())
