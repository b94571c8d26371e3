"""``python -m paper_2405_00698_b200 {run,resume,bench,export-mesh} ...``:
the reference CLI (voxevo_main.cpp) over this build (runner.main)."""
import sys

from .runner import main

sys.exit(main())
