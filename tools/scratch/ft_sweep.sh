for cfg in "4 6" "3 6" "2 6" "3 3" "2 10"; do
  set -- $cfg
  make -s -C paper_1201_2936_b200/csrc clean; make -s -C paper_1201_2936_b200/csrc EXTRA="-DSH_FTEST_MINB=$1 -DF_LOCAL_N=$2" || { echo fail; continue; }
  echo "MINB=$1 F_LOCAL=$2 $(grep -A2 k_f_test paper_1201_2936_b200/csrc/build.log | grep -o 'Used [0-9]* registers\|[0-9]* bytes spill stores' | tr '\n' ' ')"
  timeout 300 python tools/filter_probe.py 2>&1 | grep -o "uniform-ball [0-9]*\|'filter': [0-9.]*" | tr '\n' ' '; echo
done
