cd $GRAFT_REPO_ROOT
for v in ${P3V:-old sb4}; do timeout 60 ./build/p3/$v; done
