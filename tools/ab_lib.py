"""A/B two builds of libmpcb200 on one box: python tools/ab_lib.py <lib.so> <tool args...>
(points the binding at the given shared object, then runs one_ozaki_rect's body)"""
import os
import runpy
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_16013_b200 import _lib  # noqa: E402

_lib.LIB_PATH = os.path.abspath(sys.argv[1])
sys.argv = [sys.argv[2]] + sys.argv[3:]
runpy.run_path(sys.argv[0], run_name="__main__")
