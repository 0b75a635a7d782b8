for e in 1e-12 0; do ORACLE_EPS=$e timeout 1700 python tools/expt_r22.py c2:all c2z:all c3:0 c3:10 c4:11 c4z:11 c4:0 c5:11 2>&1 | grep -v Warn; done > gpurun_out/r22b.log 2>&1
