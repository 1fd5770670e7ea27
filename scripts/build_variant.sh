# Build a side library with makespan.cu (or $FILE) constants replaced (ablation / sweeps):
#   bash scripts/build_variant.sh NAME 'sed-expression' -> variants/libNAME.so
set -e
name=$1; expr=$2
d=/tmp/variant_$name
rm -rf $d && mkdir -p $d/paper_2602_23685_b200
cp -r /root/repo/paper_2602_23685_b200/csrc $d/paper_2602_23685_b200/
cp -r /root/repo/include $d/
sed -i "$expr" $d/paper_2602_23685_b200/csrc/${FILE:-makespan.cu}
mkdir -p /root/repo/variants
nvcc $EXTRA -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC -shared \
     -I$d/include $d/paper_2602_23685_b200/csrc/*.cu -o /root/repo/variants/lib$name.so
rm -rf $d
