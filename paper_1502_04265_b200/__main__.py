"""``python -m paper_1502_04265_b200 ...``: the piecy CLI (cli.py) on the GPU."""
import sys

from .cli import main

sys.exit(main())
