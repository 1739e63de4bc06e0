# Phase traces of several library builds: bash tools/trace_ab.sh SAMPLES lib1.so lib2.so ...
cd $GRAFT_REPO_ROOT
S=$1; shift
for lib in "$@"; do
  n=$(basename $lib .so)
  VPB_LIB_PATH=$PWD/$lib timeout 300 python tools/smpc_trace.py --flush --samples $S > gpurun_out/tr_${n}_$S.json 2>/dev/null
done
