for w in c2 c3; do timeout 900 python scripts/diag_fullsize.py $w 1500 > gpurun_out/diag_$w.json 2> gpurun_out/diag_$w.err; tail -2 gpurun_out/diag_$w.err; head -30 gpurun_out/diag_$w.json; done
