"""python -m paper_2203_02507_b200 <subcommand> ...: the `fpm` command line (cli.py)."""
import sys

from .cli import main

sys.exit(main())
