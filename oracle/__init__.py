"""TEST INFRASTRUCTURE ONLY: CPU restatement of the reference hot path (oracle.cpp, oracle.py) and of its
solver (solver_oracle.py). Imported by tests/, __graft_entry__.smoke() and bench.py's CPU legs only."""
