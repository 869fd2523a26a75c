"""CPU oracle (test infrastructure only; see fc2t2_oracle.py)."""
