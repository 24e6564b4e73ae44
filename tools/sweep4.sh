set -u
T="timeout -s KILL 400 python tools/tune.py"
$T --S 64 --grid 'HF_GA=1,0;HF_TW=8,6,12;HF_SPLIT=8,4' 2>&1
$T --S 64 --sets 'HF_GA=1 HF_SC=32 HF_TW=8 HF_SPLIT=8|HF_GA=1 HF_SC=32 HF_TW=16 HF_SPLIT=16|HF_GA=1 HF_TW=8 HF_SPLIT=8 HF_SLEEP_MAX=32|HF_GA=1 HF_TW=8 HF_SPLIT=8 HF_SLEEP_MAX=256' 2>&1
$T --S 256 --grid 'HF_GA=1,0;HF_TW=8,16' 2>&1
$T --S 16 --grid 'HF_GA=1,0;HF_TW=8,16,24' 2>&1
