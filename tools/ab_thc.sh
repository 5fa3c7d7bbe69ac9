# A/B timing of library variants: bash tools/ab_thc.sh name1 lib1 name2 lib2 ...
while [ $# -gt 1 ]; do
  echo "== $1"; GRADCOMP_B200_LIB=$2 FUSED_ONLY=1 python tools/time_thc.py; shift 2
done
