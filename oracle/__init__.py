"""fp64 CPU oracle for the A^2ATS decode-time retrieval path.

TEST INFRASTRUCTURE ONLY: importable from tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  Never from the product
package.  See a2ats_oracle.py for citations.
"""
from .a2ats_oracle import *  # noqa: F401,F403
