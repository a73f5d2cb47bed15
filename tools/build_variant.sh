# Builds an A/B variant of the product library into build_ab/NAME/ (git-
# ignored, travels to the GPU box): bash tools/build_variant.sh NAME "-DFLAG=.." ["NVCC-ONLY FLAGS"]
set -e
name=$1; extra=$2; nvextra=$3
make -j8 BUILD=build_ab/$name/obj LIB=build_ab/$name/libpdsim_gpu.so EXTRA="$extra" NVEXTRA="$nvextra" build_ab/$name/libpdsim_gpu.so
