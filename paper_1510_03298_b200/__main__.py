"""``python -m paper_1510_03298_b200 fit|predict ...`` (the reference's kronglm CLI)."""
import sys

from .cli import main

sys.exit(main())
