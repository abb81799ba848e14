set -e
cd paper_2012_08099_b200/csrc
for v in "0 0 5" "1 0 5" "0 1 5" "0 0 6" "0 1 6"; do
  set -- $v
  rm -f _build/project_stream.o ../libdpm_b200.so
  make -s EXTRA="-DDPM_ZX_FMA=$1 -DDPM_EARLY_RELEASE=$2 -DDPM_STAGES_U16=$3" > /dev/null 2>&1
  cd ../..
  echo "ZX_FMA=$1 EARLY=$2 STAGES=$3"
  python tools/time_project.py 2>&1 | grep -E "1024\^3 u16 K6|1024\^3 u16 K4|cfg3-like"
  cd paper_2012_08099_b200/csrc
done
