# SF1 timing with / without the ignore pass (diagnostics)
for m in 0 1; do
  if [ $m = 1 ]; then export SFK_NO_SF1_IGNORE=1; else unset SFK_NO_SF1_IGNORE; fi
  echo "no_ignore=$m"
  timeout 300 python tools/one_build.py sf1 1.0 3 2>&1 | grep "rep 2"
  timeout 600 python tools/one_build.py sf1rec 1.2 2 2>&1 | grep "rep 1"
done
