"""CPU oracle (test infrastructure): see vgicp_oracle.py.  Imported only by tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline legs."""
