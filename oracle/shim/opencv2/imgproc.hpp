// OpenCV compile stub (see imgcodecs.hpp). TEST INFRASTRUCTURE ONLY.
#pragma once
#include "opencv2/imgcodecs.hpp"
