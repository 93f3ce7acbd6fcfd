for W in ${@:-C2 C3 C5d12 C5d16}; do
  python tools/ab_lib.py paper_1111_1373_b200/libspectree_b200_old.so $W
  python tools/ab_lib.py paper_1111_1373_b200/libspectree_b200.so $W
done
