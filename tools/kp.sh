for v in "$@"; do LJMD_LIB=$PWD/paper_1704_03329_b200/libljmd_$v.so python tools/kprof.py 10 2>&1 | grep -v Warning; done
