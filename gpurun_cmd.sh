T="timeout 60"
for F in 32; do for d in powerlaw uniform; do
(cd abold && $T python ../tools/time_cfgs.py 16777216 1048576 $F f32 $d -- '' | sed 's/^/OLD /')
$T python tools/time_cfgs.py 16777216 1048576 $F f32 $d -- '' | sed 's/^/NEW /'
done; done
(cd abold && $T python ../tools/time_cfgs.py 16777216 1048576 64 bf16 powerlaw -- '' | sed 's/^/OLD /')
$T python tools/time_cfgs.py 16777216 1048576 64 bf16 powerlaw -- '' | sed 's/^/NEW /'
(cd abold && $T python ../tools/time_cfgs.py 16777216 1048576 16 f32 uniform -- '' | sed 's/^/OLD /')
$T python tools/time_cfgs.py 16777216 1048576 16 f32 uniform -- '' '{"variant":3}' | sed 's/^/NEW /'
