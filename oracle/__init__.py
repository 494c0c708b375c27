"""CPU oracle (test infrastructure only; see ncgp_oracle.py header)."""
