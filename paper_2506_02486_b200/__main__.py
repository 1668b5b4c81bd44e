"""`python -m paper_2506_02486_b200 ...` == the reference's `diomp-run ...`."""

import sys

from .cli import main

sys.exit(main())
