"""``python -m paper_2405_00698_b200 run.json [--resume checkpoint.json]``:
run / resume an evolution from a reference run-config file (runner.main)."""
import sys

from .runner import main

sys.exit(main())
