for v in 2.0 8.0 1000.0; do
  make -s -C paper_1201_2936_b200/csrc clean; make -s -C paper_1201_2936_b200/csrc EXTRA="-DSH_FGRID_SLACK=$v" || continue
  echo "SLACK=$v"; timeout 300 python tools/filter_probe.py 2>&1 | grep -o "uniform-ball [0-9]*\|unit-cube [0-9]*\|.filter.: [0-9.]*\|G=[0-9]*" | tr "\n" " "; echo
done
