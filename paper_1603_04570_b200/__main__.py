"""python -m paper_1603_04570_b200 {run,mesh-study,eps-study,verify} --config FILE (cli.py)"""
import sys

from .cli import main

sys.exit(main())
