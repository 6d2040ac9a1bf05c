for ex in "" "-DSH_R1_FAKEATOMIC"; do
  make -s -C paper_1201_2936_b200/csrc clean; make -s -C paper_1201_2936_b200/csrc EXTRA="-DF_LOCAL_N=6 $ex" || { echo "build fail"; continue; }
  echo "EXTRA=$ex"
  for r in 1 2; do timeout 200 python tools/round_probe.py uniform-disk 2>&1 | grep "round 1:"; done
done
