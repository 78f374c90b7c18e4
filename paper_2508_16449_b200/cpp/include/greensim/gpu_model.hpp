// Forwarder: the reference header name, served by the B200 drop-in API.
#pragma once
#include "gsb_greensim.hpp"
