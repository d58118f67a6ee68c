"""CPU oracle (test infrastructure only; see fmm_oracle.py header)."""
