for cfg in "2" "3" "4"; do
  make -s -C paper_1201_2936_b200/csrc clean; make -s -C paper_1201_2936_b200/csrc EXTRA="-DSH_R1_MINB=$cfg" || { echo "build fail $cfg"; continue; }
  echo "MINB=$cfg $(grep -A2 'k_round1ILi2' paper_1201_2936_b200/csrc/build.log | grep -o 'Used [0-9]* registers\|[0-9]* bytes spill stores' | tr '\n' ' ')"
  for r in 1 2 3; do timeout 200 python tools/round_probe.py uniform-disk 2>&1 | grep "round [123]:" | tr '\n' ' '; echo; done
done
