for v in ng ns ngs; do echo "== $v"; SPMVB_LIB=$PWD/paper_1612_00530_b200/libspmvcomp_b200_$v.so python tests/hybrid_probe.py 2>&1 | grep "round 1"; done
