# round-end evidence + ncu of the current build in one call
#   gpurun -- 'bash tools/sess_final2.sh TAG'
set -u
T=$1
bash tools/sess_ncu.sh ${T}_ncu
bash tools/sess_final.sh ${T}_fin
