# build timing check (diagnostics)
for a in 1.0; do timeout 300 python tools/one_build.py sff $a 3 2>&1 | grep "rep 2"; done
timeout 300 python tools/one_build.py cu 1.0 3 2>&1 | grep "rep 2"
timeout 300 python tools/one_build.py sf1 1.0 3 2>&1 | grep "rep 2"
