"""TEST INFRASTRUCTURE ONLY: CPU restatement of the reference hot path (oracle.cpp, oracle.py) and of its
solver (solver_oracle.py), plus the reference's own filter-path sources compiled in place against an Eigen
stand-in (ref_capi.cpp, eigen_standin/, ref.py -> _ref/). Imported by tests/, __graft_entry__.smoke() and
bench.py's CPU legs only."""
