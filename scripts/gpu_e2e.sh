for v in "" _old; do echo "lib [$v]"; LPD_LIBRARY=$PWD/paper_2207_01016_b200/liblpd_nystrom$v.so timeout 300 python scripts/e2e_probe.py c2 2>&1 | tail -6; done
