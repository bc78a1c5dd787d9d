run() { tag=$1; shift; timeout 60 env "$@" > gpurun_out/dbg5_$tag.log 2>&1; echo "$tag rc $?"; tail -4 gpurun_out/dbg5_$tag.log; }
run a_2slab_n128 python profiles/dev/slab_debug.py 32 16 128 2 15 40
run b_3slab_n64 python profiles/dev/slab_debug.py 30 16 64 3 16 40
run c_3slab_n128_single NO2=1 python profiles/dev/slab_debug.py 30 16 128 3 16 40
run d_3slab_n128_src5 python profiles/dev/slab_debug.py 30 16 128 3 5 40
run e_2slab_n128_src3 python profiles/dev/slab_debug.py 32 16 128 2 3 40
