"""ORACLE package — test infrastructure only (see harl_oracle.py header)."""
