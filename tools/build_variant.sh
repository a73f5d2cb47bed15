# Builds an A/B variant of the product library into build_ab/NAME/ (git-
# ignored, travels to the GPU box): bash tools/build_variant.sh NAME "-DFLAG=.."
set -e
name=$1; extra=$2
make -j8 BUILD=build_ab/$name/obj LIB=build_ab/$name/libpdsim_gpu.so EXTRA="$extra" build_ab/$name/libpdsim_gpu.so
