for v in 3 6 10; do
  make -s -C paper_1201_2936_b200/csrc clean; make -s -C paper_1201_2936_b200/csrc EXTRA="-DF_LOCAL_N=$v" || exit 1
  echo "F_LOCAL=$v"; timeout 200 python tools/filter_probe.py 2>&1 | grep -v "trace\|rounds ms"
done
