# Checked build of libtnb (device-side bounds checks + bounded stream-K spins, TNB_DCHECK in
# csrc/common.cuh) -- run the GPU suite against it with TNB_LIB_PATH:
#   bash tools/build_checked.sh && TNB_LIB_PATH=$PWD/paper_2401_01921_b200/build/libtnb_checked.so python -m pytest tests -m gpu
set -e
cd "$(dirname "$0")/.."
python -m paper_2401_01921_b200._build -DTNB_CHECKED=1 --out=$PWD/paper_2401_01921_b200/build/libtnb_checked.so
