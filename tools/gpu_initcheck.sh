timeout 900 compute-sanitizer --tool initcheck --kernel-regex kns=rsvdb --print-limit 20 python tools/initcheck_c2.py 8192 > gpurun_out/initcheck.txt 2>&1; echo rc=$?
head -80 gpurun_out/initcheck.txt
