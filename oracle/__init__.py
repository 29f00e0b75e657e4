"""Float64 CPU oracle for the HGF hot path — TEST INFRASTRUCTURE ONLY (see hgf_oracle.py header).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this package.  It shares no code with paper_1803_00005_b200/.
"""
from .hgf_oracle import *  # noqa: F401,F403
from .hgf_oracle import MODE_GF, MODE_HGF, hgf_weights  # noqa: F401
