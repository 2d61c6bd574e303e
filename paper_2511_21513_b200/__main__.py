"""python -m paper_2511_21513_b200 ... (the reference's ``intattn`` command, cli.py)."""
import sys

from .cli import main

sys.exit(main())
