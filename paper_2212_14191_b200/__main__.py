"""`python -m paper_2212_14191_b200 ...` runs the CLI (ref `python -m rnsckks.cli`)."""
import sys

from .cli import main

sys.exit(main())
