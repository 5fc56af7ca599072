"""CPU oracle for the Katz query path -- test infrastructure only (see katz_oracle.py)."""
