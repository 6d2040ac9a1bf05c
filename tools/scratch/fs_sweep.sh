for v in 64 256 1024; do
  make -s -C paper_1201_2936_b200/csrc clean; make -s -C paper_1201_2936_b200/csrc EXTRA="-DSH_FAC_SEEDS=$v" || continue
  echo "SEEDS=$v"; timeout 200 python tools/facet_probe.py 2>&1 | cut -c1-120
done
