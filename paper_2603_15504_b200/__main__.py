"""`python -m paper_2603_15504_b200 ...` runs the conic-pdhg command line."""

from .cli import main

raise SystemExit(main())
