"""INT8 tensor-core issue rate as a function of the MMA N (diagnostics for the
Ozaki kernel, which issues N = 144 (DD) / 96 (TD, QD) MMAs): run as
for n in 256 192 144 128 96 64; do MPC_INT8_PEAK_N=$n python tools/probe_int8_n.py; done"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_16013_b200 import device  # noqa: E402

print("N =", os.environ.get("MPC_INT8_PEAK_N", "256"), "->", round(device.int8_peak() / 1e12, 1), "TOP/s")
