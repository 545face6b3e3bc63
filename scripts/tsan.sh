# ThreadSanitizer build of libconveyor's host code + the native threading driver
# (tests/native/tsan_driver.cpp).  `bash scripts/tsan.sh build` here (cross-compiles), then
# `bash scripts/tsan.sh run` on a B200 (gpurun).
set -e
R=$(cd "$(dirname "$0")/.." && pwd)
mkdir -p "$R/build"
if [ "$1" = "build" ]; then
  nvcc -gencode arch=compute_100a,code=sm_100a -O1 -g -std=c++17 -Xcompiler -fPIC,-fsanitize=thread -shared \
       -o "$R/build/libconveyor_tsan.so" "$R/paper_2406_00059_b200/csrc/engine.cu" "$R/paper_2406_00059_b200/csrc/runtime.cpp" -ldl -Xcompiler -fsanitize=thread
  g++ -std=c++17 -O1 -g -fsanitize=thread -I "$R/include" -I /usr/local/cuda/include "$R/tests/native/tsan_driver.cpp" \
      -o "$R/build/tsan_driver" -L "$R/build" -lconveyor_tsan -L /usr/local/cuda/lib64 -lcudart \
      -Wl,-rpath,"\$ORIGIN" -Wl,-rpath,/usr/local/cuda/lib64 -lpthread
  echo built
else
  TSAN_OPTIONS="halt_on_error=1 second_deadlock_stack=1" setarch "$(uname -m)" -R "$R/build/tsan_driver"
fi
