for v in 0 3 6 12; do
  make -s -C paper_1201_2936_b200/csrc clean; make -s -C paper_1201_2936_b200/csrc EXTRA="-DSH_F_EXTRA=$v" || continue
  echo "F_EXTRA=$v"; timeout 300 python tools/filter_probe.py 2>&1 | grep -o "uniform-ball [0-9]*\|unit-cube [0-9]*\|.filter.: [0-9.]*\|fallback=[0-9]*\|queries=[0-9]*" | tr "\n" " "; echo
done
timeout 200 python tools/quick_parity.py | tail -1
