#!/bin/bash
set -e
timeout 300 tools/micro/hostread_0
timeout 300 tools/micro/hostread_4000
