S="6530,512,512,0,0 6530,512,512,0,0,1 6530,512,512,0,1 6530,512,512,0,1,1 6530,512,2048,0,0,1 6530,512,2048,0,1"
echo "== default"; python tools/gemm_shapes.py $S
echo "== BN128"; MTK_GEMM_BN=128 python tools/gemm_shapes.py $S
echo "== no3d"; MTK_GEMM_NO_3D=1 python tools/gemm_shapes.py $S
echo "== pair minM 512"; MTK_GEMM_PAIR_MINM=512 python tools/gemm_shapes.py $S
