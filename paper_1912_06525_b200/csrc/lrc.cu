// lrc.cu -- placeholder until the LRC path lands
#include "driver.cuh"
